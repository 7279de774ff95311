"""B200-native base64 codec (arXiv 1910.05109, Mula & Lemire) -- Python binding.

Thin argument marshalling over the C ABI in ``include/b64gpu.h``
(``libb64gpu.so``, hand-written sm_100a kernels).  torch supplies device memory
and streams only; every step of encode / decode runs in the library's kernels.
There is no CPU fallback: the calls raise if the library is missing or the
tensors are not CUDA uint8 tensors.

    enc = encode(x)                      # x: uint8 CUDA tensor -> chars
    out, err = decode(enc)               # err = -1 or first invalid offset (R7)
    out, info = decode_async(enc)        # no host sync; info = int64[3] (err, status, out_len)
    enc, off = encode_batch(x, in_off)   # BASELINE.json configs[3]
"""
from __future__ import annotations

import ctypes
from typing import Optional, Tuple

import torch

from . import _lib
from ._lib import Alphabet, B64Error, ERR_NONE, ST_BADCHAR, ST_BADPAD, ST_LENGTH, ST_NONCANON, ST_OK  # noqa: F401

__all__ = [
    "Alphabet", "B64Error", "alphabet", "lenient_of", "standard", "url", "encoded_len", "decoded_len_max", "encode", "decode",
    "decode_async", "decode_chunk", "decode_finalize", "encode_batch", "decode_batch", "encode_batch_offsets",
    "decode_batch_offsets", "BatchContext", "DecodeContext", "decode_consume", "launch_count", "HostPipeline", "new_info", "decode_unpadded", "decode_ws",
    "encode_group", "decode_group", "codec_group", "codec_group_fused", "EncodeStream", "DecodeStream",
    "ERR_NONE",
]


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _check_t(t, name: str, dtype, device=None, need: Optional[int] = None) -> None:
    """A contiguous CUDA tensor of `dtype` (on `device` if given) with at least `need` elements;
    anything else would hand the kernels a host pointer or an undersized buffer."""
    if not isinstance(t, torch.Tensor) or t.dtype != dtype or not t.is_cuda or not t.is_contiguous():
        raise B64Error(f"{name} must be a contiguous {dtype} CUDA tensor")
    if device is not None and t.device != torch.device(device):
        raise B64Error(f"{name} is on {t.device}, expected {device}")
    if need is not None and t.numel() < need:
        raise B64Error(f"{name} too small: {t.numel()} < {need} elements")


def _check_u8(t, name: str, device=None, need: Optional[int] = None) -> None:
    _check_t(t, name, torch.uint8, device, need)


def _check_i64(t, name: str, device=None, need: Optional[int] = None) -> None:
    _check_t(t, name, torch.int64, device, need)


class _On:
    """Device guard + stream order for one call on `stream` (default: the current stream).

    The library launches on `stream`; the wrappers allocate and initialise their scratch on the
    current stream.  When the two differ, `stream` waits for the current stream right before
    every launch (reading `sp`), so those fills -- and the caller's producers -- are done before
    the kernels run; internally allocated tensors are marked as used on `stream` (owns), and
    join() makes the current stream wait for `stream` before a host read of a result."""

    def __init__(self, device, stream: Optional[torch.cuda.Stream] = None):
        self.dev = torch.device(device)
        self.guard = torch.cuda.device(self.dev)
        self.stream = stream

    def __enter__(self):
        self.guard.__enter__()
        self.cur = torch.cuda.current_stream(self.dev)
        self.s = self.stream if self.stream is not None else self.cur
        self.other = self.s.cuda_stream != self.cur.cuda_stream
        return self

    @property
    def sp(self):
        """The launch stream handle, ordered after everything queued on the current stream."""
        if self.other:
            self.s.wait_stream(self.cur)
        return ctypes.c_void_p(self.s.cuda_stream)

    def owns(self, *ts) -> None:
        if self.other:
            for t in ts:
                if t is not None:
                    t.record_stream(self.s)

    def join(self) -> None:
        if self.other:
            self.cur.wait_stream(self.s)

    def __exit__(self, *exc):
        return self.guard.__exit__(*exc)


# ------------------------------------------------------------------ alphabets

def alphabet(chars: bytes, pad: bytes = b"=", lenient: bool = False) -> Alphabet:
    """Validate a 64-char alphabet + pad (R4); returns the by-value table struct.
    lenient=True sets B64_ALPHA_LENIENT (R16) for every decode with it."""
    if len(chars) != 64 or len(pad) != 1:
        raise B64Error("alphabet needs 64 chars and a 1-byte pad")
    a = Alphabet()
    bad = ctypes.c_int(0)
    rc = _lib.lib().b64_alphabet_init(ctypes.byref(a), bytes(chars), pad, ctypes.byref(bad))
    if rc != 0:
        raise B64Error(f"invalid alphabet: {_lib.ERRORS.get(rc, rc)} at index {bad.value}")
    return lenient_of(a) if lenient else a


def lenient_of(a: Alphabet) -> Alphabet:
    """A copy of `a` with B64_ALPHA_LENIENT set (R16: non-zero trailing bits before
    the padding are dropped instead of rejected)."""
    b = Alphabet()
    ctypes.pointer(b)[0] = a
    _lib.check(_lib.lib().b64_alphabet_set_flags(ctypes.byref(b), _lib.ALPHA_LENIENT), "b64_alphabet_set_flags")
    return b


def standard() -> Alphabet:
    return _lib.lib().b64_alphabet_standard().contents


def url() -> Alphabet:
    return _lib.lib().b64_alphabet_url().contents


def _alpha(a: Optional[Alphabet]):
    return ctypes.byref(a if a is not None else standard())


def encoded_len(n: int) -> int:
    return int(_lib.lib().b64_encoded_len(n))


def decoded_len_max(m: int) -> int:
    return int(_lib.lib().b64_decoded_len_max(m))


# ------------------------------------------------------------------ single stream

def encode(x: torch.Tensor, a: Optional[Alphabet] = None, out: Optional[torch.Tensor] = None,
           stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Encode bytes to base64 chars with '=' padding (b64_encode)."""
    _check_u8(x, "x")
    n = x.numel()
    m = encoded_len(n)
    with _On(x.device, stream) as on:
        if out is None:
            out = torch.empty(m, dtype=torch.uint8, device=x.device)
            on.owns(out)
        else:
            _check_u8(out, "out", x.device, m)
        _lib.check(_lib.lib().b64_encode(_ptr(x), n, _ptr(out), _alpha(a), on.sp), "b64_encode")
    return out if out.numel() == m else out[:m]


def new_info(device=None) -> torch.Tensor:
    """A zeroed device int64[3] for decode_async: (err_off, status, out_len)."""
    return torch.zeros(3, dtype=torch.int64, device=device if device is not None else "cuda")


class DecodeContext:
    """Device context of b64_decode_fused (B64_DECODE_CTX_BYTES): with it, decode_async is ONE
    kernel launch (no initialisation, no finalize launch).  Calls sharing a context must be
    ordered (one context per stream)."""

    def __init__(self, device=None, stream: Optional[torch.cuda.Stream] = None):
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        with _On(dev, stream) as on:
            self.buf = torch.empty(_lib.DECODE_CTX_BYTES, dtype=torch.uint8, device=dev)
            on.owns(self.buf)
            _lib.check(_lib.lib().b64_decode_ctx_init(_ptr(self.buf), on.sp), "b64_decode_ctx_init")


def decode_async(t: torch.Tensor, a: Optional[Alphabet] = None, out: Optional[torch.Tensor] = None,
                 info: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None,
                 ctx: Optional[DecodeContext] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Validating decode (b64_decode_ex, or b64_decode_fused with a DecodeContext) without a
    host sync.

    Returns (out, info) where info is a device int64[3]: (err_off, status, out_len).
    A caller-provided info must come from new_info() (the status is written as an
    int32 into the low half of info[1]; the high half must stay zero)."""
    _check_u8(t, "t")
    m = t.numel()
    cap = decoded_len_max(m)
    with _On(t.device, stream) as on:
        if out is None:
            out = torch.empty(max(cap, 1), dtype=torch.uint8, device=t.device)
            on.owns(out)
        else:
            _check_u8(out, "out", t.device, cap)
        if info is None:
            info = new_info(t.device)
            on.owns(info)
        else:
            _check_i64(info, "info", t.device, 3)
        ip = info.data_ptr()
        if ctx is not None:
            _check_u8(ctx.buf, "ctx", t.device)
            _lib.check(_lib.lib().b64_decode_fused(_ptr(t), m, _ptr(out), _alpha(a), ctypes.c_void_p(ip),
                                                   ctypes.c_void_p(ip + 8), ctypes.c_void_p(ip + 16), _ptr(ctx.buf),
                                                   on.sp), "b64_decode_fused")
        else:
            _lib.check(_lib.lib().b64_decode_ex(_ptr(t), m, _ptr(out), _alpha(a), ctypes.c_void_p(ip),
                                                ctypes.c_void_p(ip + 8), ctypes.c_void_p(ip + 16), on.sp),
                       "b64_decode_ex")
    return out, info


_CTX_CACHE = {}  # (device index, stream handle) -> DecodeContext, for the synchronous decode()


def _stream_ctx(dev: torch.device, stream: Optional[torch.cuda.Stream]) -> DecodeContext:
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    key = (dev.index, s.cuda_stream)
    ctx = _CTX_CACHE.get(key)
    if ctx is None:
        ctx = _CTX_CACHE[key] = DecodeContext(dev, stream=s)
    return ctx


def decode(t: torch.Tensor, a: Optional[Alphabet] = None, out: Optional[torch.Tensor] = None,
           stream: Optional[torch.cuda.Stream] = None, ctx: Optional[DecodeContext] = None) -> Tuple[torch.Tensor, int]:
    """Validating decode.  Returns (decoded bytes, err_off); err_off = -1 when valid.
    Forces one 24-byte device->host read of (err_off, status, out_len).  One kernel launch:
    the call is synchronous, so a context cached per (device, stream) can serve every call
    on that stream (b64_decode_fused)."""
    if ctx is None:
        ctx = _stream_ctx(t.device, stream)
    out, info = decode_async(t, a, out=out, stream=stream, ctx=ctx)
    with _On(t.device, stream) as on:
        on.join()
        err, _, olen = info.tolist()
    return out[:olen], err


def decode_unpadded(t: torch.Tensor, a: Optional[Alphabet] = None, out: Optional[torch.Tensor] = None,
                    stream: Optional[torch.cuda.Stream] = None) -> Tuple[torch.Tensor, int]:
    """Padding-optional validating decode (b64_decode_unpadded, R13).
    Returns (decoded bytes, err_off); err_off = -1 when valid."""
    _check_u8(t, "t")
    m = t.numel()
    cap = int(_lib.lib().b64_decoded_len_max_unpadded(m))
    if cap < 0:
        raise B64Error("B64_ELENGTH: text length is 1 more than a multiple of 4")
    with _On(t.device, stream) as on:
        if out is None:
            out = torch.empty(max(cap, 1), dtype=torch.uint8, device=t.device)
            on.owns(out)
        else:
            _check_u8(out, "out", t.device, cap)
        info = new_info(t.device)
        on.owns(info)
        ip = info.data_ptr()
        _lib.check(_lib.lib().b64_decode_unpadded(_ptr(t), m, _ptr(out), _alpha(a), ctypes.c_void_p(ip),
                                                  ctypes.c_void_p(ip + 8), ctypes.c_void_p(ip + 16), on.sp),
                   "b64_decode_unpadded")
        on.join()
        err, _, olen = info.tolist()
    return out[:olen], err


def decode_ws(t: torch.Tensor, a: Optional[Alphabet] = None, out: Optional[torch.Tensor] = None,
              workspace: Optional[torch.Tensor] = None,
              stream: Optional[torch.cuda.Stream] = None) -> Tuple[torch.Tensor, int]:
    """Whitespace-skipping validating decode (b64_decode_ws, R14): MIME-style line
    breaks and blanks are ignored; err_off is a position in the ORIGINAL text (-1 = valid)."""
    _check_u8(t, "t")
    m = t.numel()
    cap = decoded_len_max(m)
    need = int(_lib.lib().b64_decode_ws_workspace_bytes(m))
    with _On(t.device, stream) as on:
        if out is None:
            out = torch.empty(max(cap, 1), dtype=torch.uint8, device=t.device)
            on.owns(out)
        else:
            _check_u8(out, "out", t.device, cap)
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(need, dtype=torch.uint8, device=t.device)
            on.owns(workspace)
        else:
            _check_u8(workspace, "workspace", t.device)
        info = new_info(t.device)
        on.owns(info)
        ip = info.data_ptr()
        _lib.check(_lib.lib().b64_decode_ws(_ptr(t), m, _ptr(out), _alpha(a), _ptr(workspace), workspace.numel(),
                                            ctypes.c_void_p(ip), ctypes.c_void_p(ip + 8), ctypes.c_void_p(ip + 16),
                                            on.sp), "b64_decode_ws")
        on.join()
        err, _, olen = info.tolist()
    return out[:olen], err


def decode_chunk(t: torch.Tensor, base_offset: int, is_final: bool, err_cell: torch.Tensor,
                 a: Optional[Alphabet] = None, out: Optional[torch.Tensor] = None,
                 out_len: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Shard-aware decode (b64_decode_chunk): lowers err_cell (int64[1], init ERR_NONE) with the
    packed first error (global_pos << 3 | status)."""
    _check_u8(t, "t")
    _check_i64(err_cell, "err_cell", t.device, 1)
    if out_len is not None:
        _check_i64(out_len, "out_len", t.device, 1)
    m = t.numel()
    cap = decoded_len_max(m)
    with _On(t.device, stream) as on:
        if out is None:
            out = torch.empty(max(cap, 1), dtype=torch.uint8, device=t.device)
            on.owns(out)
        else:
            _check_u8(out, "out", t.device, cap)
        _lib.check(_lib.lib().b64_decode_chunk(_ptr(t), m, _ptr(out), _alpha(a), base_offset, 1 if is_final else 0,
                                               _ptr(err_cell), _ptr(out_len), on.sp), "b64_decode_chunk")
    return out


def decode_finalize(err_cell: torch.Tensor, err_off: torch.Tensor, status: Optional[torch.Tensor] = None,
                    stream: Optional[torch.cuda.Stream] = None) -> None:
    """Packed error word -> (err_off = -1 | position, status) on the device."""
    _check_i64(err_cell, "err_cell", None, 1)
    _check_i64(err_off, "err_off", err_cell.device, 1)
    if status is not None:
        _check_t(status, "status", torch.int32, err_cell.device, 1)
    with _On(err_cell.device, stream) as on:
        _lib.check(_lib.lib().b64_decode_finalize(_ptr(err_cell), _ptr(err_off), _ptr(status), on.sp),
                   "b64_decode_finalize")


# ------------------------------------------------------------------ grouped launches

class _NoOn:
    def owns(self, *ts) -> None:
        pass


def _enc_items(xs, alphabets, outs, dev=None, on=None):
    k = len(xs)
    dev = dev if dev is not None else (xs[0].device if xs else None)
    on = on if on is not None else _NoOn()
    al = alphabets if isinstance(alphabets, (list, tuple)) else [alphabets] * k
    al = [a if a is not None else standard() for a in al]
    lens = [encoded_len(x.numel()) for x in xs]
    if outs is None:
        outs = [torch.empty(max(m, 1), dtype=torch.uint8, device=dev) for m in lens]
        on.owns(*outs)
    items = (_lib.EncodeItem * max(k, 1))()
    for i, (x, o) in enumerate(zip(xs, outs)):
        _check_u8(x, "x", dev)
        _check_u8(o, "out", dev, lens[i])
        items[i] = _lib.EncodeItem(x.data_ptr(), x.numel(), o.data_ptr(), ctypes.pointer(al[i]))
    return items, [o[:m] for m, o in zip(lens, outs)]


def _dec_items(ts, alphabets, outs, cells, bases, finals, dev=None, on=None):
    k = len(ts)
    dev = dev if dev is not None else ts[0].device
    on = on if on is not None else _NoOn()
    al = alphabets if isinstance(alphabets, (list, tuple)) else [alphabets] * k
    al = [a if a is not None else standard() for a in al]
    caps = [decoded_len_max(t.numel()) for t in ts]
    if outs is None:
        outs = [torch.empty(max(c, 1), dtype=torch.uint8, device=dev) for c in caps]
        on.owns(*outs)
    if cells is None:
        cells = torch.full((k,), ERR_NONE, dtype=torch.int64, device=dev)
        on.owns(cells)
    else:
        _check_i64(cells, "cells", dev, k)
    items = (_lib.DecodeItem * max(k, 1))()
    for i, (t, o) in enumerate(zip(ts, outs)):
        _check_u8(t, "t", dev)
        _check_u8(o, "out", dev, caps[i])
        items[i] = _lib.DecodeItem(t.data_ptr(), t.numel(), o.data_ptr(), ctypes.pointer(al[i]),
                                   0 if bases is None else bases[i], 1 if finals is None else int(finals[i]), 0,
                                   cells[i:].data_ptr())
    return items, outs, cells


def _finalize_n(cells, k, dev, on):
    err = torch.empty(k, dtype=torch.int64, device=dev)
    st = torch.empty(k, dtype=torch.int32, device=dev)
    on.owns(err, st)
    _lib.check(_lib.lib().b64_decode_finalize_n(_ptr(cells), k, _ptr(err), _ptr(st), on.sp),
               "b64_decode_finalize_n")
    return err, st


def encode_group(xs, alphabets=None, outs=None, stream: Optional[torch.cuda.Stream] = None):
    """Encode several independent device buffers with one kernel per group of 8 (b64_encode_group).
    alphabets: one Alphabet for all, or a list; returns the list of outputs."""
    dev = xs[0].device
    with _On(dev, stream) as on:
        items, outs = _enc_items(xs, alphabets, outs, dev, on)
        _lib.check(_lib.lib().b64_encode_group(items, len(xs), on.sp), "b64_encode_group")
    return outs


def decode_group(ts, alphabets=None, outs=None, cells: Optional[torch.Tensor] = None, bases=None, finals=None,
                 stream: Optional[torch.cuda.Stream] = None):
    """Validating decode of several device buffers, one kernel per group of 8 (b64_decode_group).
    Returns (outs, err_off int64[k] device tensor, status int32[k] device tensor)."""
    dev = ts[0].device
    with _On(dev, stream) as on:
        items, outs, cells = _dec_items(ts, alphabets, outs, cells, bases, finals, dev, on)
        _lib.check(_lib.lib().b64_decode_group(items, len(ts), on.sp), "b64_decode_group")
        err, st = _finalize_n(cells, len(ts), dev, on)
    return outs, err, st


def codec_group_fused(xs, ts, enc_alphabets=None, dec_alphabets=None, enc_outs=None, dec_outs=None,
                      cells: Optional[torch.Tensor] = None, ticket: Optional[torch.Tensor] = None,
                      err: Optional[torch.Tensor] = None, status: Optional[torch.Tensor] = None,
                      stream: Optional[torch.cuda.Stream] = None):
    """b64_codec_group_fused: up to 8 encodes + 8 decodes (fast-path aligned) in ONE launch whose
    last CTA also writes err/status and resets `cells` (ERR_NONE) and `ticket` (0) -- pass the
    same cells/ticket to back-to-back calls and no set-up launch is needed.  Returns
    (encoded list, decoded list, err_off int64[len(ts)], status int32[len(ts)])."""
    dev = (xs[0] if xs else ts[0]).device
    k = max(len(ts), 1)
    with _On(dev, stream) as on:
        eitems, eouts = _enc_items(xs, enc_alphabets, enc_outs, dev, on)
        if ts:
            ditems, douts, cells = _dec_items(ts, dec_alphabets, dec_outs, cells, None, None, dev, on)
        else:
            ditems, douts = (_lib.DecodeItem * 1)(), []
        if ticket is None:
            ticket = torch.zeros(1, dtype=torch.int32, device=dev)
            on.owns(ticket)
        else:
            _check_t(ticket, "ticket", torch.int32, dev, 1)
        if err is None:
            err = torch.empty(k, dtype=torch.int64, device=dev)
            on.owns(err)
        else:
            _check_i64(err, "err", dev, len(ts))
        if status is None:
            status = torch.empty(k, dtype=torch.int32, device=dev)
            on.owns(status)
        else:
            _check_t(status, "status", torch.int32, dev, len(ts))
        _lib.check(_lib.lib().b64_codec_group_fused(eitems, len(xs), ditems, len(ts), _ptr(err), _ptr(status),
                                                    _ptr(ticket), on.sp), "b64_codec_group_fused")
    return eouts, douts, err[: len(ts)], status[: len(ts)]


def codec_group(xs, ts, enc_alphabets=None, dec_alphabets=None, enc_outs=None, dec_outs=None,
                cells: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None):
    """Independent encodes of xs and validating decodes of ts, ONE kernel per group of up to 8 + 8
    (b64_codec_group).  Returns (encoded list, decoded list, err_off int64[len(ts)] or None,
    status int32[len(ts)] or None)."""
    dev = (xs[0] if xs else ts[0]).device
    with _On(dev, stream) as on:
        eitems, eouts = _enc_items(xs, enc_alphabets, enc_outs, dev, on)
        if ts:
            ditems, douts, cells = _dec_items(ts, dec_alphabets, dec_outs, cells, None, None, dev, on)
        else:
            ditems, douts = (_lib.DecodeItem * 1)(), []
        _lib.check(_lib.lib().b64_codec_group(eitems, len(xs), ditems, len(ts), on.sp), "b64_codec_group")
        if not ts:
            return eouts, douts, None, None
        err, st = _finalize_n(cells, len(ts), dev, on)
    return eouts, douts, err, st


# ------------------------------------------------------------------ decode -> consumer (L2-resident ring)

def decode_consume(t: torch.Tensor, consumer, a: Optional[Alphabet] = None, ring_bytes: int = 64 << 20,
                   ring: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None):
    """b64_decode_consume: decode `t` chunk by chunk into an L2-sized device ring and call
    consumer(chunk, out_offset) after each chunk -- chunk is a uint8 view of the ring holding
    that chunk's decoded bytes, out_offset their position in the whole output; the consumer
    queues its own GPU work on the current stream, which reads the bytes while they are in L2
    (SURVEY.md Sec. 8(f) f3).  Returns (err_off, out_len) after the device finished."""
    _check_u8(t, "t")
    dev = t.device
    with _On(dev, stream) as on:
        if ring is None:
            ring = torch.empty(ring_bytes, dtype=torch.uint8, device=dev)
            on.owns(ring)
        else:
            _check_u8(ring, "ring", dev)
        info = new_info(dev)
        on.owns(info)
        base = ring.data_ptr()
        errors = []

        def _cb(d_chunk, n, off, user, s_):
            try:
                k = int(d_chunk) - base
                with torch.cuda.stream(on.s):
                    consumer(ring[k: k + n], off)
            except Exception as e:  # noqa: BLE001 -- re-raised after the C loop returns
                errors.append(e)

        cb = _lib.CONSUMER_FN(_cb)
        ip = info.data_ptr()
        _lib.check(_lib.lib().b64_decode_consume(_ptr(t), t.numel(), _ptr(ring), ring.numel(), _alpha(a), cb, None,
                                                 ctypes.c_void_p(ip), ctypes.c_void_p(ip + 8),
                                                 ctypes.c_void_p(ip + 16), on.sp), "b64_decode_consume")
        if errors:
            raise errors[0]
        on.join()
        err, _, olen = info.tolist()
    return err, olen


# ------------------------------------------------------------------ streaming (carry between calls)

class _StreamBase:
    def __init__(self, a: Optional[Alphabet], device, stream: Optional[torch.cuda.Stream]):
        self.a = _alpha(a)
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        # the CUDA stream is fixed once per object: every call of one stream must be ordered
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.dev)
        self.st = _lib.Stream()

    def out_len(self, n: int) -> int:
        """Bytes / chars the next update with a piece of n writes (b64_stream_update_len)."""
        return int(_lib.lib().b64_stream_update_len(ctypes.byref(self.st), n))

    def end_len(self) -> int:
        """Capacity the end call needs (b64_stream_end_len)."""
        return int(_lib.lib().b64_stream_end_len(ctypes.byref(self.st)))

    def _out(self, out, k, on):
        if out is None:
            out = torch.empty(max(k, 1), dtype=torch.uint8, device=self.dev)
            on.owns(out)
        else:
            _check_u8(out, "out", self.dev, k)
        return out


class EncodeStream(_StreamBase):
    """Encode input that arrives in pieces of any length (b64_encode_stream_*).

    update(x) returns the chars completed so far (a view of a fresh or given buffer);
    end() returns the padded tail.  The concatenation of every returned piece equals
    encode(concatenation of the inputs).  All calls run on the CUDA stream fixed at
    construction (default: the current stream then).

    overlap=True: b64_encode_stream_begin_ex with B64_STREAM_OVERLAP (contract as
    DecodeStream's: every piece's input written before construction, nothing else on the
    stream writes a piece's input or output until end(), inputs and outputs disjoint)."""

    def __init__(self, a: Optional[Alphabet] = None, device=None, stream: Optional[torch.cuda.Stream] = None,
                 overlap: bool = False):
        super().__init__(a, device, stream)
        with _On(self.dev, self.stream) as on:
            self.carry = torch.zeros(8, dtype=torch.uint8, device=self.dev)
            on.owns(self.carry)
            _lib.check(_lib.lib().b64_encode_stream_begin_ex(ctypes.byref(self.st), _ptr(self.carry),
                                                             _lib.STREAM_OVERLAP if overlap else 0, on.sp),
                       "b64_encode_stream_begin_ex")

    def update(self, x: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        _check_u8(x, "x", self.dev)
        with _On(self.dev, self.stream) as on:
            out = self._out(out, self.out_len(x.numel()), on)
            n_out = ctypes.c_int64(0)
            _lib.check(_lib.lib().b64_encode_stream_update(ctypes.byref(self.st), _ptr(x), x.numel(), _ptr(out),
                                                           self.a, ctypes.byref(n_out), on.sp),
                       "b64_encode_stream_update")
        return out[: n_out.value]

    def end(self, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        with _On(self.dev, self.stream) as on:
            out = self._out(out, self.end_len(), on)
            n_out = ctypes.c_int64(0)
            _lib.check(_lib.lib().b64_encode_stream_end(ctypes.byref(self.st), _ptr(out), self.a,
                                                        ctypes.byref(n_out), on.sp), "b64_encode_stream_end")
        return out[: n_out.value]


class DecodeStream(_StreamBase):
    """Validating decode of text that arrives in pieces of any length (b64_decode_stream_*).

    update(t) returns the bytes of the quads completed so far (the last 1-4 chars are
    held back); end() returns (tail bytes tensor, info) with info = int64[3] device tensor
    (err_off, status, out_len) for the whole concatenated text, exactly as decode_async.
    All calls run on the CUDA stream fixed at construction.

    overlap=True: b64_decode_stream_begin_ex with B64_STREAM_OVERLAP -- each piece's
    bulk starts while the previous piece drains; the caller guarantees every piece's
    input is written before construction, nothing else on the stream writes any
    piece's input or output until end(), and inputs do not overlap outputs
    (include/b64gpu.h)."""

    def __init__(self, a: Optional[Alphabet] = None, device=None, stream: Optional[torch.cuda.Stream] = None,
                 overlap: bool = False):
        super().__init__(a, device, stream)
        with _On(self.dev, self.stream) as on:
            self.carry = torch.zeros(8, dtype=torch.uint8, device=self.dev)
            self.cell = torch.empty(1, dtype=torch.int64, device=self.dev)
            on.owns(self.carry, self.cell)
            _lib.check(_lib.lib().b64_decode_stream_begin_ex(ctypes.byref(self.st), _ptr(self.carry), _ptr(self.cell),
                                                             _lib.STREAM_OVERLAP if overlap else 0, on.sp),
                       "b64_decode_stream_begin_ex")

    def update(self, t: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        _check_u8(t, "t", self.dev)
        with _On(self.dev, self.stream) as on:
            out = self._out(out, self.out_len(t.numel()), on)
            n_out = ctypes.c_int64(0)
            _lib.check(_lib.lib().b64_decode_stream_update(ctypes.byref(self.st), _ptr(t), t.numel(), _ptr(out),
                                                           self.a, ctypes.byref(n_out), on.sp),
                       "b64_decode_stream_update")
        return out[: n_out.value]

    def end(self, out: Optional[torch.Tensor] = None):
        with _On(self.dev, self.stream) as on:
            out = self._out(out, self.end_len(), on)
            info = new_info(self.dev)
            on.owns(info)
            ip = info.data_ptr()
            n_out = ctypes.c_int64(0)
            _lib.check(_lib.lib().b64_decode_stream_end(ctypes.byref(self.st), _ptr(out), self.a, ctypes.c_void_p(ip),
                                                        ctypes.c_void_p(ip + 8), ctypes.c_void_p(ip + 16),
                                                        ctypes.byref(n_out), on.sp), "b64_decode_stream_end")
        return out[: n_out.value], info


# ------------------------------------------------------------------ host buffers (overlapped pipeline)

class HostPipeline:
    """Device workspaces + three streams for b64_encode_host / b64_decode_host.

    Chunks of a host buffer rotate through 3 device buffers: H2D copy, kernel
    and D2H copy of consecutive chunks overlap (both PCIe directions busy).
    Calls alternate between two workspaces and are issued with
    B64_HOST_CALLER_ORDERED: a call only waits (on its H2D stream) for the end
    of the call before last -- the previous user of its workspace -- so
    back-to-back sync=False calls overlap each other too.  join() makes the
    current stream wait for everything issued; sync=True calls join and
    synchronise."""

    def __init__(self, chunk_bytes: int = 16 << 20, device=None):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.device = dev
        self.ws_bytes = int(_lib.lib().b64_host_workspace_bytes(chunk_bytes))
        self.ws = [torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev) for _ in range(2)]
        self.done = [None, None]  # event at the end of the last call on each workspace
        self.turn = 0
        self.streams = [torch.cuda.Stream(device=dev) for _ in range(3)]
        self.info = new_info(dev)

    def _sp(self):
        return [ctypes.c_void_p(s.cuda_stream) for s in self.streams]

    def _begin(self):
        """Order a new call: after the caller's queued work, and after the previous user of the
        workspace it gets.  Returns the workspace."""
        w = self.turn
        self.turn ^= 1
        cur = torch.cuda.current_stream(self.device)
        for s in self.streams:
            s.wait_stream(cur)
        if self.done[w] is not None:
            self.streams[0].wait_event(self.done[w])
        return w

    def _end(self, w):
        # the D2H stream's last copy waited for the kernels, which waited for the H2D copies; it
        # also waits for the rest of the compute stream (the decode finalize) before the mark
        self.streams[2].wait_stream(self.streams[1])
        ev = torch.cuda.Event()
        ev.record(self.streams[2])
        self.done[w] = ev

    def join(self):
        cur = torch.cuda.current_stream(self.device)
        for s in self.streams:
            cur.wait_stream(s)

    def encode(self, x: torch.Tensor, a: Optional[Alphabet] = None, out: Optional[torch.Tensor] = None,
               sync: bool = True) -> torch.Tensor:
        if x.is_cuda or x.dtype != torch.uint8 or not x.is_contiguous():
            raise B64Error("x must be a contiguous uint8 host tensor (pinned for overlap)")
        m = encoded_len(x.numel())
        if out is None:
            out = torch.empty(max(m, 1), dtype=torch.uint8, pin_memory=True)
        elif out.is_cuda or out.dtype != torch.uint8 or not out.is_contiguous() or out.numel() < m:
            raise B64Error(f"out must be a contiguous uint8 host tensor of >= {m} bytes")
        with torch.cuda.device(self.device):
            w = self._begin()
            _lib.check(_lib.lib().b64_encode_host_ex(_ptr(x), x.numel(), _ptr(out), _alpha(a), _ptr(self.ws[w]),
                                                     self.ws_bytes, *self._sp(), _lib.HOST_CALLER_ORDERED),
                       "b64_encode_host_ex")
            self._end(w)
            if sync:
                self.join()
                torch.cuda.current_stream(self.device).synchronize()
        return out[:m]

    def decode(self, t: torch.Tensor, a: Optional[Alphabet] = None, out: Optional[torch.Tensor] = None,
               sync: bool = True, info: Optional[torch.Tensor] = None):
        """Returns (host bytes, err_off) when sync, else (host buffer, device info int64[3] = (err_off,
        status in the low half of [1], out_len) -- a fresh one per call unless `info` is given;
        overlapped calls must not share it).  The exact output length comes from the device."""
        if t.is_cuda or t.dtype != torch.uint8 or not t.is_contiguous():
            raise B64Error("t must be a contiguous uint8 host tensor (pinned for overlap)")
        m = t.numel()
        cap = decoded_len_max(m)
        if out is None:
            out = torch.empty(max(cap, 1), dtype=torch.uint8, pin_memory=True)
        elif out.is_cuda or out.dtype != torch.uint8 or not out.is_contiguous() or out.numel() < cap:
            raise B64Error(f"out must be a contiguous uint8 host tensor of >= {cap} bytes")
        with torch.cuda.device(self.device):
            if info is None:
                info = self.info if sync else new_info(self.device)
            else:
                _check_i64(info, "info", self.device, 3)
            w = self._begin()
            with torch.cuda.stream(self.streams[1]):
                info[1].zero_()  # the status is an int32 in the low half
            ip = info.data_ptr()
            _lib.check(_lib.lib().b64_decode_host_ex(_ptr(t), m, _ptr(out), _alpha(a), _ptr(self.ws[w]),
                                                     self.ws_bytes, ctypes.c_void_p(ip), ctypes.c_void_p(ip + 8),
                                                     ctypes.c_void_p(ip + 16), *self._sp(), _lib.HOST_CALLER_ORDERED),
                       "b64_decode_host_ex")
            self._end(w)
            if not sync:
                return out, info
            self.join()
            err, _, olen = info.tolist()
        return out[:olen], err


# ------------------------------------------------------------------ batched

def encode_batch_offsets(in_off: torch.Tensor, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Device int64[count+1] output offsets of a batch encode: exclusive scan of 4*ceil(len/3),
    computed by the library on the device (b64_encode_batch_offsets)."""
    _check_i64(in_off, "in_off", None, 1)
    with _On(in_off.device, stream) as on:
        out_off = torch.empty(in_off.numel(), dtype=torch.int64, device=in_off.device)
        on.owns(out_off)
        _lib.check(_lib.lib().b64_encode_batch_offsets(_ptr(in_off), in_off.numel() - 1, _ptr(out_off), on.sp),
                   "b64_encode_batch_offsets")
    return out_off


def decode_batch_offsets(in_off: torch.Tensor, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Device int64[count+1] output offsets of a batch decode: exclusive scan of 3*floor(len/4)
    (b64_decode_batch_offsets)."""
    _check_i64(in_off, "in_off", None, 1)
    with _On(in_off.device, stream) as on:
        out_off = torch.empty(in_off.numel(), dtype=torch.int64, device=in_off.device)
        on.owns(out_off)
        _lib.check(_lib.lib().b64_decode_batch_offsets(_ptr(in_off), in_off.numel() - 1, _ptr(out_off), on.sp),
                   "b64_decode_batch_offsets")
    return out_off


class BatchContext:
    """Device context of b64_decode_batch_fast (B64_BATCH_CTX_BYTES): enables the batched decode's
    concatenation path.  Self-resetting; calls sharing a context must be ordered (one per stream)."""

    def __init__(self, device=None, stream: Optional[torch.cuda.Stream] = None):
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        with _On(dev, stream) as on:
            self.buf = torch.empty(_lib.BATCH_CTX_BYTES, dtype=torch.uint8, device=dev)
            on.owns(self.buf)
            _lib.check(_lib.lib().b64_batch_ctx_init(_ptr(self.buf), on.sp), "b64_batch_ctx_init")


_BATCH_CTX_CACHE = {}  # (device index, stream handle) -> BatchContext


def _batch_ctx(dev: torch.device, s: torch.cuda.Stream) -> BatchContext:
    key = (dev.index, s.cuda_stream)
    ctx = _BATCH_CTX_CACHE.get(key)
    if ctx is None:
        ctx = _BATCH_CTX_CACHE[key] = BatchContext(dev, stream=s)
    return ctx


def _batch_total(out_off: torch.Tensor, on: "_On") -> int:
    on.join()
    return int(out_off[-1].item())


def encode_batch(x: torch.Tensor, in_off: torch.Tensor, a: Optional[Alphabet] = None,
                 out: Optional[torch.Tensor] = None, out_off: Optional[torch.Tensor] = None,
                 total_out: Optional[int] = None,
                 stream: Optional[torch.cuda.Stream] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Per-string padded encode of strings concatenated in x (offsets int64[count+1]).
    Returns (out, out_off) with out_off = exclusive scan of 4*ceil(len/3) (int64[count+1]).
    A caller-given out is checked against total_out (if given) or out_off[-1]."""
    _check_u8(x, "x")
    dev = x.device
    _check_i64(in_off, "in_off", dev, 1)
    count = in_off.numel() - 1
    with _On(dev, stream) as on:
        if x.numel() == 0:  # all strings empty: the C ABI still wants a valid (unread) pointer
            x = torch.empty(1, dtype=torch.uint8, device=dev)
            on.owns(x)
        if out_off is None:
            out_off = encode_batch_offsets(in_off, stream=on.s)
        else:
            _check_i64(out_off, "out_off", dev, count + 1)
        if total_out is None:
            total_out = _batch_total(out_off, on)
        if out is None:
            out = torch.empty(max(total_out, 1), dtype=torch.uint8, device=dev)
            on.owns(out)
        else:
            _check_u8(out, "out", dev, total_out)
        _lib.check(_lib.lib().b64_encode_batch(_ptr(x), _ptr(in_off), count, _ptr(out), _ptr(out_off), _alpha(a),
                                               on.sp), "b64_encode_batch")
    return out, out_off


def decode_batch(t: torch.Tensor, in_off: torch.Tensor, a: Optional[Alphabet] = None,
                 out: Optional[torch.Tensor] = None, out_off: Optional[torch.Tensor] = None,
                 total_out: Optional[int] = None, stream: Optional[torch.cuda.Stream] = None,
                 index_base: int = 0, first_bad: Optional[torch.Tensor] = None,
                 ctx: Optional[BatchContext] = None, fast: bool = True):
    """Per-string validating decode.  Returns (out, out_off, status int32, err_off int64
    (relative, -1 = ok), out_len int64); out_off = exclusive scan of 3*(len//4).
    first_bad (device int64[1], caller-initialised, e.g. ERR_NONE): lowered to index_base + the
    index of the first failing string.  fast (default): b64_decode_batch_fast with `ctx` (or
    a context cached per device and stream) -- the concatenation path when the batch is
    eligible; fast=False: b64_decode_batch_ex (the per-string kernel only).  Bytes of a
    string's slot after its out_len are unspecified."""
    _check_u8(t, "t")
    dev = t.device
    _check_i64(in_off, "in_off", dev, 1)
    count = in_off.numel() - 1
    if first_bad is not None:
        _check_i64(first_bad, "first_bad", dev, 1)
    with _On(dev, stream) as on:
        if t.numel() == 0:  # all strings empty: the C ABI still wants a valid (unread) pointer
            t = torch.empty(1, dtype=torch.uint8, device=dev)
            on.owns(t)
        if out_off is None:
            out_off = decode_batch_offsets(in_off, stream=on.s)
        else:
            _check_i64(out_off, "out_off", dev, count + 1)
        if total_out is None:
            total_out = _batch_total(out_off, on)
        if out is None:
            out = torch.empty(max(total_out, 1), dtype=torch.uint8, device=dev)
            on.owns(out)
        else:
            _check_u8(out, "out", dev, total_out)
        status = torch.empty(max(count, 1), dtype=torch.int32, device=dev)
        err = torch.empty(max(count, 1), dtype=torch.int64, device=dev)
        olen = torch.empty(max(count, 1), dtype=torch.int64, device=dev)
        on.owns(status, err, olen)
        cbuf = None
        if fast:
            cbuf = (ctx if ctx is not None else _batch_ctx(dev, on.s)).buf
            _check_u8(cbuf, "ctx", dev)
        _lib.check(_lib.lib().b64_decode_batch_fast(_ptr(t), _ptr(in_off), count, _ptr(out), _ptr(out_off), _alpha(a),
                                                    _ptr(status), _ptr(err), _ptr(olen), index_base,
                                                    _ptr(first_bad) if first_bad is not None else None, _ptr(cbuf),
                                                    on.sp), "b64_decode_batch_fast")
    return out, out_off, status[:count], err[:count], olen[:count]


def launch_count() -> int:
    """Kernels this process launched through the library (host-side counter)."""
    return int(_lib.lib().b64_launch_count())


def build_info() -> str:
    return _lib.lib().b64_build_info().decode()
