"""Scalar CPU oracle for the base64 codec -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_1910_05109_b200`` never imports it; the two share no
code.

The arithmetic lives in ``oracle.c`` (plain C, one byte / one quad at a time,
each function citing the PAPER.md passage it follows).  This module is only
ctypes marshalling over numpy arrays plus the alphabet strings the paper
prints:

* standard alphabet -- PAPER.md:239 (Sec. 3.1 step 2; Table 1's body is
  missing from the source, reading R1);
* base64url -- PAPER.md:93 ('+' and '/' replaced by '-' and '_').
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# PAPER.md:239, verbatim.
STANDARD = b"ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/"
# '+' -> '-', '/' -> '_'.
URL = STANDARD[:62] + b"-_"
PAD = ord("=")

ST_OK, ST_BADCHAR, ST_BADPAD, ST_NONCANON, ST_LENGTH = 0, 1, 2, 3, 4


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc into liboracle.so (the checker, not the product)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        U8 = ctypes.c_uint8
        L.oracle_alphabet_check.argtypes = [P, U8, ctypes.POINTER(ctypes.c_int)]
        L.oracle_alphabet_check.restype = ctypes.c_int
        L.oracle_encoded_len.argtypes = [I64]
        L.oracle_encoded_len.restype = I64
        L.oracle_encode.argtypes = [P, I64, P, P, U8]
        L.oracle_encode.restype = I64
        L.oracle_decode.argtypes = [P, I64, P, P, U8, ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.oracle_decode.restype = ctypes.c_int
        L.oracle_decode_unpadded.argtypes = [P, I64, P, P, U8, ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.oracle_decode_unpadded.restype = ctypes.c_int
        L.oracle_decode_ws.argtypes = [P, I64, P, P, U8, ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.oracle_decode_ws.restype = ctypes.c_int
        for nm in ("oracle_decode_lenient", "oracle_decode_unpadded_lenient", "oracle_decode_ws_lenient"):
            getattr(L, nm).argtypes = [P, I64, P, P, U8, ctypes.POINTER(I64), ctypes.POINTER(I64)]
            getattr(L, nm).restype = ctypes.c_int
        L.oracle_decode_batch_opt.argtypes = [P, P, I64, P, P, P, U8, ctypes.c_int, P, P, P]
        L.oracle_decode_batch_opt.restype = None
        L.oracle_encode_batch.argtypes = [P, P, I64, P, P, P, U8]
        L.oracle_encode_batch.restype = None
        L.oracle_decode_batch.argtypes = [P, P, I64, P, P, P, U8, P, P, P]
        L.oracle_decode_batch.restype = None
        _lib = L
    return _lib


def _u8(x) -> np.ndarray:
    if isinstance(x, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(x), dtype=np.uint8)
    a = np.ascontiguousarray(x)
    assert a.dtype == np.uint8
    return a


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _alpha(chars: bytes) -> np.ndarray:
    a = _u8(chars)
    assert a.size == 64
    return a


def alphabet_check(chars: bytes, pad: int = PAD):
    """Returns (code, bad_index); code 0 ok, -3 duplicate, -4 non-ASCII, -5 pad in alphabet."""
    a = _alpha(chars)
    bad = ctypes.c_int(0)
    r = lib().oracle_alphabet_check(_ptr(a), pad, ctypes.byref(bad))
    return r, bad.value


def encoded_len(n: int) -> int:
    return int(lib().oracle_encoded_len(n))


def encode(data, chars: bytes = STANDARD, pad: int = PAD) -> np.ndarray:
    x = _u8(data)
    out = np.empty(encoded_len(x.size) + 1, dtype=np.uint8)  # +1: never pass a NULL-ish empty buffer
    m = lib().oracle_encode(_ptr(x) if x.size else None, x.size, _ptr(out), _ptr(_alpha(chars)), pad)
    return out[:m]


def decode(text, chars: bytes = STANDARD, pad: int = PAD, lenient: bool = False):
    """Returns (bytes ndarray of the exact prefix, err_off, status).  lenient: reading R16
    (non-zero trailing bits before the padding are dropped instead of rejected)."""
    t = _u8(text)
    out = np.empty(3 * (t.size // 4) + 1, dtype=np.uint8)
    ol = ctypes.c_int64(0)
    eo = ctypes.c_int64(0)
    f = lib().oracle_decode_lenient if lenient else lib().oracle_decode
    st = f(_ptr(t) if t.size else None, t.size, _ptr(out), _ptr(_alpha(chars)), pad,
                             ctypes.byref(ol), ctypes.byref(eo))
    return out[: ol.value], eo.value, st


def decode_unpadded(text, chars: bytes = STANDARD, pad: int = PAD, lenient: bool = False):
    """Padding-optional decode (reading R13; + R16 when lenient).  Returns (exact prefix bytes,
    err_off, status)."""
    t = _u8(text)
    out = np.empty(3 * (t.size // 4) + 3, dtype=np.uint8)
    ol = ctypes.c_int64(0)
    eo = ctypes.c_int64(0)
    f = lib().oracle_decode_unpadded_lenient if lenient else lib().oracle_decode_unpadded
    st = f(_ptr(t) if t.size else None, t.size, _ptr(out), _ptr(_alpha(chars)), pad,
                                      ctypes.byref(ol), ctypes.byref(eo))
    return out[: ol.value], eo.value, st


def decode_ws(text, chars: bytes = STANDARD, pad: int = PAD, lenient: bool = False):
    """Whitespace-skipping decode (reading R14; + R16 when lenient).  Returns (exact prefix
    bytes, err_off in the original text, status)."""
    t = _u8(text)
    out = np.empty(3 * (t.size // 4) + 1, dtype=np.uint8)
    ol = ctypes.c_int64(0)
    eo = ctypes.c_int64(0)
    f = lib().oracle_decode_ws_lenient if lenient else lib().oracle_decode_ws
    st = f(_ptr(t) if t.size else None, t.size, _ptr(out), _ptr(_alpha(chars)), pad,
                                ctypes.byref(ol), ctypes.byref(eo))
    return out[: ol.value], eo.value, st


def encode_unpadded(data, chars: bytes = STANDARD, pad: int = PAD) -> np.ndarray:
    """encode() with the trailing '=' dropped (the length law without padding)."""
    t = encode(data, chars, pad)
    n = _u8(data).size
    return t[: t.size - (3 - n % 3) % 3]


def encode_batch(data, in_off, chars: bytes = STANDARD, pad: int = PAD):
    """Returns (concatenated output, out_off)."""
    x = _u8(data)
    in_off = np.ascontiguousarray(in_off, dtype=np.int64)
    count = in_off.size - 1
    lens = np.diff(in_off)
    out_off = np.zeros(count + 1, dtype=np.int64)
    np.cumsum(4 * ((lens + 2) // 3), out=out_off[1:])
    out = np.empty(int(out_off[-1]) + 1, dtype=np.uint8)
    xs = x if x.size else np.zeros(1, np.uint8)
    lib().oracle_encode_batch(_ptr(xs), _ptr(in_off), count, _ptr(out), _ptr(out_off), _ptr(_alpha(chars)), pad)
    return out[: out_off[-1]], out_off


def decode_batch(text, in_off, chars: bytes = STANDARD, pad: int = PAD, lenient: bool = False):
    """Returns (out buffer laid out at out_off = scan(3*len//4), out_off, status, err_off, out_len)."""
    t = _u8(text)
    in_off = np.ascontiguousarray(in_off, dtype=np.int64)
    count = in_off.size - 1
    lens = np.diff(in_off)
    out_off = np.zeros(count + 1, dtype=np.int64)
    np.cumsum(3 * (lens // 4), out=out_off[1:])
    out = np.zeros(int(out_off[-1]) + 1, dtype=np.uint8)
    status = np.zeros(max(count, 1), dtype=np.int32)
    err = np.zeros(max(count, 1), dtype=np.int64)
    olen = np.zeros(max(count, 1), dtype=np.int64)
    ts = t if t.size else np.zeros(1, np.uint8)
    lib().oracle_decode_batch_opt(_ptr(ts), _ptr(in_off), count, _ptr(out), _ptr(out_off), _ptr(_alpha(chars)), pad,
                                  int(lenient), _ptr(status), _ptr(err), _ptr(olen))
    return out[: out_off[-1]], out_off, status[:count], err[:count], olen[:count]
