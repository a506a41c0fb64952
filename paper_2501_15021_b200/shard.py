"""Multi-GPU sharding of the AKVQ-VL hot path (BJ:5).

Every unit u = b * Hkv + h (batch row x KV head) is independent: saliency is
per unit (R2), quantization is per unit, and decode attention of unit u reads
only unit u's cache.  So the units are split into contiguous ranges, one per
rank, and each rank allocates, fills and attends over its own caches with no
communication.  The one exchange step is the all-gather of the attention
outputs, which this module does with
``torch.distributed.all_gather_into_tensor`` (NCCL over NVLink on the GPU box,
gloo in the CPU tests).

Host logic only: no arithmetic of the method lives here.
"""
from __future__ import annotations

from typing import List, Optional, Tuple

import torch


def unit_range(U: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced range [lo, hi) of the b-major units owned by `rank`.

    The first U % world ranks get one extra unit, so sizes differ by at most one.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if U < 0:
        raise ValueError("negative unit count")
    base, extra = divmod(U, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def unit_ranges(U: int, world: int) -> List[Tuple[int, int]]:
    return [unit_range(U, world, r) for r in range(world)]


def max_local_units(U: int, world: int) -> int:
    return (U + world - 1) // world


class OutputGather:
    """All-gather of per-rank outputs [.., U_local, g, d] into [.., U, g, d].

    Ranks with fewer units (U % world != 0) pad their slice to the largest
    slice so the collective is a single equal-sized ``all_gather_into_tensor``;
    the padding is dropped when the result is unpacked.  Buffers are allocated
    once and reused every step.  `lead` is the shape of leading dims (e.g. the
    layer count when a whole step's outputs are gathered at once).
    """

    def __init__(self, U: int, world: int, rank: int, g: int, d: int,
                 lead: Tuple[int, ...] = (), dtype=torch.float32, device="cpu",
                 group=None):
        self.U, self.world, self.rank = U, world, rank
        self.ranges = unit_ranges(U, world)
        self.Um = max_local_units(U, world)
        self.lo, self.hi = self.ranges[rank]
        self.group = group
        self.lead = tuple(lead)
        self.even = U % world == 0
        self.send = torch.zeros(self.lead + (self.Um, g, d), dtype=dtype, device=device)
        self.recv = torch.empty((world,) + self.lead + (self.Um, g, d), dtype=dtype, device=device)
        self.out = torch.empty(self.lead + (U, g, d), dtype=dtype, device=device)

    def local_view(self) -> torch.Tensor:
        """Where this rank writes its own outputs ([.., U_local, g, d])."""
        return self.send[..., : self.hi - self.lo, :, :]

    def gather(self, async_op: bool = False):
        """Launch the all-gather; returns the work handle when async_op."""
        import torch.distributed as dist
        return dist.all_gather_into_tensor(self.recv.view(-1), self.send.view(-1),
                                           group=self.group, async_op=async_op)

    def result(self) -> torch.Tensor:
        """[.., U, g, d] in global unit order (after the gather completed)."""
        nl = len(self.lead)
        if self.even and nl == 0:
            return self.recv.view(self.U, *self.recv.shape[-2:])
        for r, (lo, hi) in enumerate(self.ranges):
            self.out[..., lo:hi, :, :] = self.recv[r][..., : hi - lo, :, :]
        return self.out


def gather_outputs(local: torch.Tensor, U: int, world: int, rank: int,
                   group: Optional[object] = None) -> torch.Tensor:
    """One-shot convenience: gather [U_local, g, d] slices into [U, g, d]."""
    g, d = local.shape[-2:]
    og = OutputGather(U, world, rank, g, d, lead=tuple(local.shape[:-3]), dtype=local.dtype,
                      device=local.device, group=group)
    og.local_view().copy_(local)
    og.gather()
    return og.result().clone()
