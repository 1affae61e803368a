"""Host <-> device plumbing for the drop-in entry points: the reference's
callers hand over pageable numpy arrays (int64 columns, float64 values,
core.py:130-137) and expect numpy results, and a pageable cudaMemcpy moves
~11 GB/s where the link does 55.  Large transfers therefore go through a small
pool of pinned buffers: uploads are copied into a pinned ring by several host
threads (numpy releases the GIL) while the previous chunk is in flight, and
batch results land in a pooled pinned array instead of freshly faulted pages.

torch is used for pinned allocation, streams and events only."""

from __future__ import annotations

import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_LOCK = threading.Lock()
_FREE: list = []  # pinned uint8 tensors not in use
_KEEP = 4  # buffers kept for reuse (the largest ones)
_CHUNK = 64 << 20  # upload ring chunk
_PARTS = 8  # host threads per chunk copy
_COPIERS = ThreadPoolExecutor(max_workers=_PARTS, thread_name_prefix="ds-hostio")
MIN_BYTES = 64 << 20  # below this the plain path is as fast
MAX_POOLED = 16 << 30  # largest result array taken from the pool (pinning more starves the host)


def available() -> bool:
    try:
        import torch
    except ImportError:
        return False
    return torch.cuda.is_available()


def take_pinned(nbytes: int):
    """A pinned uint8 tensor of at least `nbytes` (reused when one is free)."""
    import torch

    with _LOCK:
        best = None
        for i, t in enumerate(_FREE):
            # same size class only: a ring chunk must not take the one big result buffer
            if nbytes <= t.numel() <= 4 * nbytes and (best is None or t.numel() < _FREE[best].numel()):
                best = i
        if best is not None:
            return _FREE.pop(best)
    return torch.empty(int(nbytes), dtype=torch.uint8, pin_memory=True)


def give_pinned(t) -> None:
    with _LOCK:
        _FREE.append(t)
        _FREE.sort(key=lambda x: -x.numel())
        del _FREE[_KEEP:]


def clear() -> None:
    with _LOCK:
        _FREE.clear()


def _copy_parts(dst: np.ndarray, src: np.ndarray) -> None:
    n = dst.shape[0]
    step = (n + _PARTS - 1) // _PARTS
    step = (step + 4095) & ~4095

    def part(p):
        a, b = p * step, min(n, (p + 1) * step)
        if a < b:
            np.copyto(dst[a:b], src[a:b])

    list(_COPIERS.map(part, range(_PARTS)))


def upload(arr: np.ndarray, device: int):
    """`arr` (C-contiguous host array) as a device tensor of the same dtype,
    through the pinned ring."""
    import torch

    tdt = {np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64,
           np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}[arr.dtype]
    dev = torch.empty(arr.shape, dtype=tdt, device=f"cuda:{device}")
    src = arr.reshape(-1).view(np.uint8)
    dst = dev.reshape(-1).view(torch.uint8)
    nbytes = src.shape[0]
    ring = [take_pinned(_CHUNK) for _ in range(3)]
    try:
        stream = torch.cuda.Stream(device=device)
        events = [torch.cuda.Event() for _ in ring]
        for i, off in enumerate(range(0, nbytes, _CHUNK)):
            slot = i % len(ring)
            if i >= len(ring):
                events[slot].synchronize()  # the chunk that used this buffer has left it
            ln = min(_CHUNK, nbytes - off)
            _copy_parts(ring[slot].numpy()[:ln], src[off:off + ln])
            with torch.cuda.stream(stream):
                dst[off:off + ln].copy_(ring[slot][:ln], non_blocking=True)
                events[slot].record(stream)
        stream.synchronize()
    finally:
        for b in ring:
            give_pinned(b)
    return dev
