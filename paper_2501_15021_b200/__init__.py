"""B200-native (sm_100a) AKVQ-VL hot path (arXiv 2501.15021).

The CUDA library ``libakvq.so`` (C-ABI, ``include/akvq.h``) is loaded lazily by
``paper_2501_15021_b200.akvq``; importing this package does not touch the GPU,
so host-side helpers (``synth``) work on CPU-only machines.
"""
__all__ = ["akvq", "synth"]
