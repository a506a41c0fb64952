"""Seeded synthetic inputs for the AKVQ-VL hot path (shared by tests and bench).

This module holds NONE of the method's arithmetic (no rotation, saliency,
quantization or attention).  It only draws the inputs the paper's workloads
would feed the path -- post-RoPE K/V rows, token-type masks, accumulated
attention column sums and decode-step q/k/v -- with the shapes, value
distributions and structure of BASELINE.json's configs (BJ:7-11; recipe in
DESIGN.md "Synthetic inputs").  MileBench prompts are not in the
container; these synthetic caches stand in for them.

Every value is a pure function of (workload seed, layer, unit, tensor kind,
step, element index) through a counter-based hash, computed with integer
torch ops that give identical results on CPU and CUDA.  So a sampled unit
generated on the CPU for the oracle equals the same unit generated on the GPU,
and sharded runs see exactly the data of the unsharded run.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import torch

TEXT, VISION = 1, 0
_M32 = 0xFFFFFFFF


@dataclass(frozen=True)
class Workload:
    name: str
    n_layers: int
    batch: int
    hq: int
    hkv: int
    d: int
    G: int
    R: int
    top_k: int
    dtype: str                      # "bf16" | "fp16"
    segments: Tuple[Tuple[int, int], ...]   # (type, count) runs of the prompt
    tsa_layers: Tuple[int, ...]
    n_outlier_ch: int               # K outlier channels per layer
    outlier_gain: float
    fixed_outlier_ch: Tuple[int, ...] = ()  # if set, used instead of random
    pivots_fixed: Tuple[int, ...] = (0,)    # planted pivot positions
    pivots_random_vision: int = 0           # + this many random vision positions
    pivots_per_frame: bool = False          # + one random vision position per frame
    pivot_logit: float = 8.0
    decode_steps: int = 128
    seed: int = 0
    clip2: float = 0.8
    clip4: float = 1.0
    hidden: int = 4096                      # residual-stream width (NEXT-2 inputs)

    @property
    def g(self) -> int:
        return self.hq // self.hkv

    @property
    def U(self) -> int:
        return self.batch * self.hkv

    @property
    def L0(self) -> int:
        return sum(c for _, c in self.segments)

    @property
    def capacity(self) -> int:
        return self.L0 + self.decode_steps

    def kind(self, layer: int) -> int:
        """0 = TSA, 1 = PSA (Table I)."""
        return 0 if layer in self.tsa_layers else 1

    def with_batch(self, batch: int) -> "Workload":
        d = dict(self.__dict__)
        d["batch"] = batch
        d["name"] = f"{self.name.split('@')[0]}@b{batch}"
        return Workload(**d)


def _run(*parts):
    return tuple(parts)


# BJ:7 tiny: [16 T][64 V][16 T], fp16, 4 MHA heads, d 64, G 32, top-4, R 8.
TINY = Workload("tiny", 1, 1, 4, 4, 64, 32, 8, 4, "fp16",
                _run((TEXT, 16), (VISION, 64), (TEXT, 16)), (), 2, 20.0,
                fixed_outlier_ch=(3, 17), pivots_fixed=(0, 40), decode_steps=16, hidden=256)
# BJ:8 LLaVA-1.5-7B: 32 L, 32 MHA heads, d 128, [35 T][576 V][60 T] = 671.
LLAVA7B = Workload("llava7b", 32, 1, 32, 32, 128, 128, 32, 15, "bf16",
                   _run((TEXT, 35), (VISION, 576), (TEXT, 60)), (0, 1), 4, 15.0,
                   pivots_random_vision=2, decode_steps=128)
# BJ:9 batch sweep at 7B shape: [35 T]([576 V][10 T])x3[55 T] = 1848.
SWEEP = Workload("sweep", 32, 64, 32, 32, 128, 128, 32, 15, "bf16",
                 _run((TEXT, 35), *((VISION, 576), (TEXT, 10)) * 3, (TEXT, 55)),
                 (0, 1), 4, 15.0, pivots_random_vision=2, decode_steps=256)
# BJ:10 LLaVA-13B video: 40 L, 40 heads, batch 8, [35 T]([576 V][5 T])x8[125 T].
VIDEO13B = Workload("video13b", 40, 8, 40, 40, 128, 128, 64, 15, "bf16",
                    _run((TEXT, 35), *((VISION, 576), (TEXT, 5)) * 8, (TEXT, 125)),
                    (0, 1), 4, 15.0, pivots_per_frame=True, decode_steps=128, hidden=5120)
# BJ:11 Qwen2-VL-like GQA: 28 L, 28/4 heads, batch 16, [68 T]([600 V][54 T])x50.
QWEN = Workload("qwen_gqa", 28, 16, 28, 4, 128, 128, 128, 8, "bf16",
                _run((TEXT, 68), *((VISION, 600), (TEXT, 54)) * 50), (0, 1), 4, 20.0,
                pivots_random_vision=7, decode_steps=64, hidden=3584)

WORKLOADS = {w.name: w for w in (TINY, LLAVA7B, SWEEP, VIDEO13B, QWEN)}


def get(name: str) -> Workload:
    if "@b" in name:
        base, b = name.split("@b")
        return WORKLOADS[base].with_batch(int(b))
    return WORKLOADS[name]


# ------------------------------------------------------------- counter hash
def _h32(x: torch.Tensor) -> torch.Tensor:
    """lowbias32 integer finaliser on uint32 values held in int64."""
    x = x & _M32
    x = ((x ^ (x >> 16)) * 0x7FEB352D) & _M32
    x = ((x ^ (x >> 15)) * 0x846CA68B) & _M32
    return x ^ (x >> 16)


def _key(*parts: int) -> int:
    k = 0x9E3779B9
    for p in parts:
        k = int(_h32(torch.tensor([(k ^ (p & _M32)) & _M32], dtype=torch.int64))[0])
        k = (k * 0x01000193 + 0x7F4A7C15) & _M32
    return k


_KIND = {"K": 1, "V": 2, "q": 3, "k": 4, "v": 5, "attn": 6, "ch": 7, "piv": 8, "res": 9}


def _uniform_bits(keys: torch.Tensor, n: int, device) -> torch.Tensor:
    """keys [U] int64 -> [U, n] uint32-in-int64 hashes of (key, counter)."""
    ctr = torch.arange(n, dtype=torch.int64, device=device)
    return _h32(_h32(ctr[None, :] + keys[:, None]) ^ (keys[:, None] * 0x2C1B3C6D & _M32))


def normal(keys: torch.Tensor, n: int, device) -> torch.Tensor:
    """[U, n] standard normals (Box-Muller in float64) from per-row keys."""
    a = _uniform_bits(keys, 2 * n, device).view(keys.shape[0], n, 2)
    u1 = (a[..., 0].to(torch.float64) + 1.0) / 4294967296.0      # (0, 1]
    u2 = a[..., 1].to(torch.float64) / 4294967296.0              # [0, 1)
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)


def _unit_keys(w: Workload, layer: int, units: Sequence[int], kind: str, step: int,
               device) -> torch.Tensor:
    base = _key(w.seed, layer, _KIND[kind], step)
    u = torch.as_tensor(list(units), dtype=torch.int64, device=device)
    return _h32(u * 0x27D4EB2F + base)


def _dtype(w: Workload):
    return torch.bfloat16 if w.dtype == "bf16" else torch.float16


def token_types(w: Workload) -> torch.Tensor:
    """[L0] uint8, 1 = text, 0 = vision, in prompt order (BJ:7-11)."""
    return torch.cat([torch.full((c,), t, dtype=torch.uint8) for t, c in w.segments])


def outlier_channels(w: Workload, layer: int) -> List[int]:
    """Per layer, n random K channels scaled by `outlier_gain` (BJ:8, BJ:11)."""
    if w.fixed_outlier_ch:
        return list(w.fixed_outlier_ch)
    keys = torch.tensor([_key(w.seed, layer, _KIND["ch"])], dtype=torch.int64)
    h = _uniform_bits(keys, 4 * w.n_outlier_ch, "cpu")[0].tolist()
    chans: List[int] = []
    for x in h:
        c = int(x) % w.d
        if c not in chans:
            chans.append(c)
        if len(chans) == w.n_outlier_ch:
            break
    return chans


def pivot_positions(w: Workload, batch_row: int) -> List[int]:
    """Planted pivot tokens of one batch row (BJ:7-11)."""
    types = token_types(w)
    vis = torch.nonzero(types == VISION).flatten().tolist()
    piv = [p for p in w.pivots_fixed if p < w.L0]
    keys = torch.tensor([_key(w.seed, batch_row, _KIND["piv"])], dtype=torch.int64)
    h = _uniform_bits(keys, 64, "cpu")[0].tolist()
    if w.pivots_per_frame:
        # one random vision position inside each vision run (frame)
        frames, start = [], 0
        for t, c in w.segments:
            if t == VISION:
                frames.append((start, c))
            start += c
        for i, (s, c) in enumerate(frames):
            piv.append(s + int(h[i]) % c)
    else:
        want = len(w.pivots_fixed) + min(w.pivots_random_vision, len(vis))
        i = 0
        while len(piv) < want and i < len(h):
            p = vis[int(h[i]) % len(vis)]
            i += 1
            if p not in piv:
                piv.append(p)
    return piv


def _round16(x64: torch.Tensor, w: Workload) -> torch.Tensor:
    return x64.to(torch.float32).to(_dtype(w))


def layer_inputs(w: Workload, layer: int, units: Optional[Sequence[int]] = None,
                 device="cpu") -> dict:
    """Prefill inputs of one layer for the given units (default: all).

    K, V [n, L0, d] 16-bit (post-RoPE rows, N(0,1), K outlier channels x gain);
    types [n, L0] u8; colsum [n, g, L0] f32 = softmax over tokens of one random
    query row per query head with +pivot_logit at the planted pivots.
    """
    units = list(range(w.U)) if units is None else list(units)
    n, L0, d, g = len(units), w.L0, w.d, w.g
    K = normal(_unit_keys(w, layer, units, "K", 0, device), L0 * d, device).view(n, L0, d)
    V = normal(_unit_keys(w, layer, units, "V", 0, device), L0 * d, device).view(n, L0, d)
    ch = outlier_channels(w, layer)
    if ch:
        K[:, :, ch] *= w.outlier_gain
    types = token_types(w).to(device)[None, :].expand(n, L0).contiguous()
    z = normal(_unit_keys(w, layer, units, "attn", 0, device), g * L0, device).view(n, g, L0)
    for i, u in enumerate(units):
        b = u // w.hkv
        z[i, :, pivot_positions(w, b)] += w.pivot_logit
    colsum = torch.softmax(z, dim=-1).to(torch.float32)
    return dict(K=_round16(K, w), V=_round16(V, w), types=types, colsum=colsum)


def decode_inputs(w: Workload, layer: int, step: int,
                  units: Optional[Sequence[int]] = None, device="cpu") -> dict:
    """One decode step: q [n, g, d], k, v [n, d] (16-bit), types [n] (text)."""
    units = list(range(w.U)) if units is None else list(units)
    n, d, g = len(units), w.d, w.g
    q = normal(_unit_keys(w, layer, units, "q", step + 1, device), g * d, device).view(n, g, d)
    k = normal(_unit_keys(w, layer, units, "k", step + 1, device), d, device).view(n, d)
    v = normal(_unit_keys(w, layer, units, "v", step + 1, device), d, device).view(n, d)
    ch = outlier_channels(w, layer)
    if ch:
        k[:, ch] *= w.outlier_gain
    types = torch.full((n,), TEXT, dtype=torch.uint8, device=device)
    return dict(q=_round16(q, w), k=_round16(k, w), v=_round16(v, w), types=types)


def to_u16(t: torch.Tensor):
    """16-bit torch tensor -> numpy uint16 bit patterns (for the oracle)."""
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view("uint16")


def residual_inputs(w: Workload, rows: Optional[Sequence[int]] = None, device="cpu",
                    magnitude: float = 1000.0) -> torch.Tensor:
    """Residual stream [n_rows, L0, hidden] (16-bit) of the batch rows (NEXT-2).

    Background N(0,1); at each planted pivot of the row (pivot_positions) two
    fixed channels carry a massive activation (Sun et al., cited at P:209) of
    +-magnitude * (1 - 0.05 i) for the i-th pivot, so the expected pivot order
    is the planted order.  The same pivots drive colsum in layer_inputs.
    """
    rows = list(range(w.batch)) if rows is None else list(rows)
    n, L0, hd = len(rows), w.L0, w.hidden
    keys = _unit_keys(w, 0, rows, "res", 0, device)
    x = normal(keys, L0 * hd, device).view(n, L0, hd)
    ck = torch.tensor([_key(w.seed, _KIND["res"], 1)], dtype=torch.int64)
    h = _uniform_bits(ck, 2, "cpu")[0].tolist()
    chans = [int(h[0]) % hd, (int(h[0]) % hd + 1 + int(h[1]) % (hd - 1)) % hd]
    for i, b in enumerate(rows):
        for j, p in enumerate(pivot_positions(w, b)):
            m = magnitude * (1.0 - 0.05 * j)
            x[i, p, chans[0]] = m
            x[i, p, chans[1]] = -m
    return _round16(x, w)

