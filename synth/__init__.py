"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the codec's arithmetic: it only draws random
numbers.  Both sides receive the same bytes from it (or, for inputs too big to
copy, the same counter-based generator implemented again in ``synth.cu`` and
checked bit-exact against this file by ``tests/test_synth.py``).

Generator:

* byte i of stream (seed, sid) = (W[i // 8] >> 8 * (i % 8)) & 0xFF
* W[j] = mix64(key + (j + 1) * 0x9E3779B97F4A7C15), key = seed * 2**32 + sid
* mix64 = the splitmix64 finalizer.
* sid 0 = data bytes, 1 = corruption positions, 2 = corruption bytes,
  3 = string lengths (config 4), 4 = which strings get corrupted (config 4).

The generator has O(1) random access, so any shard or chunk can be produced
on its own (multi-GPU ranks, chunk-wise oracle checks).
"""
from __future__ import annotations

import math

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

SID_DATA, SID_POS, SID_BAD, SID_LEN, SID_PICK = 0, 1, 2, 3, 4


def key(seed: int, sid: int) -> int:
    return ((seed << 32) + sid) & 0xFFFFFFFFFFFFFFFF


def words(seed: int, sid: int, j0: int, count: int) -> np.ndarray:
    """W[j0 .. j0+count) as uint64."""
    with np.errstate(over="ignore"):
        j = np.arange(j0 + 1, j0 + 1 + count, dtype=np.uint64)
        z = np.uint64(key(seed, sid)) + j * GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return z


def stream_bytes(seed: int, sid: int, offset: int, n: int) -> np.ndarray:
    """Bytes [offset, offset + n) of stream (seed, sid)."""
    if n <= 0:
        return np.zeros(0, dtype=np.uint8)
    j0 = offset // 8
    j1 = (offset + n - 1) // 8
    w = words(seed, sid, j0, j1 - j0 + 1).astype("<u8")
    b = w.view(np.uint8)
    s = offset - 8 * j0
    return b[s: s + n].copy()


def data(n: int, seed: int = 0, offset: int = 0) -> np.ndarray:
    """The uniform random input bytes of every config (sid 0)."""
    return stream_bytes(seed, SID_DATA, offset, n)


def distinct_positions(k: int, m: int, seed: int = 0, sid: int = SID_POS) -> np.ndarray:
    """k distinct positions in [0, m): W[j] mod m, skipping repeats, in draw order."""
    if k > m:
        raise ValueError("k > m")
    out: list[int] = []
    seen: set[int] = set()
    j = 0
    while len(out) < k:
        need = max(64, 2 * (k - len(out)))
        w = words(seed, sid, j, need)
        j += need
        for v in (w % np.uint64(m)).tolist():
            if v not in seen:
                seen.add(v)
                out.append(v)
                if len(out) == k:
                    break
    return np.array(out, dtype=np.int64)


def bad_set(chars: bytes, pad: int = ord("=")) -> np.ndarray:
    """BAD63: the ASCII bytes that are neither alphabet chars nor the pad, ascending."""
    s = set(chars) | {pad}
    return np.array([c for c in range(128) if c not in s], dtype=np.uint8)


def corruption(k: int, m: int, chars: bytes, seed: int = 0, pad: int = ord("=")):
    """(positions, bytes): k distinct positions in [0, m) and a BAD63 byte for each."""
    pos = distinct_positions(k, m, seed)
    bad = bad_set(chars, pad)
    w = words(seed, SID_BAD, 0, k)
    return pos, bad[(w % np.uint64(bad.size)).astype(np.int64)]


def loguniform_lengths(count: int, lo: int = 1, hi: int = 65536, seed: int = 0) -> np.ndarray:
    """Config 4: L_i = min(hi, max(lo, floor(exp(u_i * ln(hi + 1))))), u_i 53-bit from sid 3."""
    w = words(seed, SID_LEN, 0, count)
    u = (w >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    L = np.floor(np.exp(u * math.log(hi + 1)))
    return np.clip(L, lo, hi).astype(np.int64)


def offsets(lengths: np.ndarray) -> np.ndarray:
    off = np.zeros(lengths.size + 1, dtype=np.int64)
    np.cumsum(lengths, out=off[1:])
    return off


def pick(count: int, frac: float, seed: int = 0) -> np.ndarray:
    """Indices i < count chosen with probability frac (sid 4), ascending."""
    w = words(seed, SID_PICK, 0, count)
    thr = np.uint64(int(frac * 2.0 ** 64) if frac < 1 else 0xFFFFFFFFFFFFFFFF)
    return np.nonzero(w < thr)[0].astype(np.int64)


# ---------------------------------------------------------------- device twin

_dev_lib = None


def _device_lib():
    global _dev_lib
    if _dev_lib is None:
        import ctypes
        import os

        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} not built (run __graft_entry__.build())")
        L = ctypes.CDLL(path)
        L.synth_fill.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                 ctypes.c_void_p]
        L.synth_fill.restype = ctypes.c_int
        _dev_lib = L
    return _dev_lib


def device_fill(t, seed: int = 0, sid: int = SID_DATA, offset: int = 0, stream=None):
    """Fill a contiguous uint8 CUDA tensor with bytes [offset, offset + numel) of stream (seed, sid)."""
    import ctypes

    import torch

    assert t.dtype == torch.uint8 and t.is_cuda and t.is_contiguous()
    s = stream if stream is not None else torch.cuda.current_stream()
    rc = _device_lib().synth_fill(ctypes.c_void_p(t.data_ptr()), t.numel(), seed, sid, offset,
                                  ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"synth_fill failed: {rc}")
    return t


def device_data(n: int, seed: int = 0, offset: int = 0, device="cuda"):
    import torch

    t = torch.empty(n, dtype=torch.uint8, device=device)
    return device_fill(t, seed, SID_DATA, offset)
