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
    "decode_async", "decode_chunk", "decode_finalize", "encode_batch", "decode_batch", "launch_count", "HostPipeline", "new_info", "decode_unpadded", "decode_ws",
    "encode_group", "decode_group", "codec_group", "codec_group_fused", "EncodeStream", "DecodeStream",
    "ERR_NONE",
]


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _check_u8(t: torch.Tensor, name: str) -> None:
    if not isinstance(t, torch.Tensor) or t.dtype != torch.uint8 or not t.is_cuda or not t.is_contiguous():
        raise B64Error(f"{name} must be a contiguous uint8 CUDA tensor")


def _check_i64(t: torch.Tensor, name: str) -> None:
    if not isinstance(t, torch.Tensor) or t.dtype != torch.int64 or not t.is_cuda or not t.is_contiguous():
        raise B64Error(f"{name} must be a contiguous int64 CUDA tensor")


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
    m = 4 * ((n + 2) // 3)  # b64_encoded_len
    if out is None:
        out = torch.empty(m, dtype=torch.uint8, device=x.device)
    else:
        _check_u8(out, "out")
        if out.numel() < m:
            raise B64Error("out too small")
    _lib.check(_lib.lib().b64_encode(_ptr(x), n, _ptr(out), _alpha(a), _stream(stream)), "b64_encode")
    return out if out.numel() == m else out[:m]


def new_info(device=None) -> torch.Tensor:
    """A zeroed device int64[3] for decode_async: (err_off, status, out_len)."""
    return torch.zeros(3, dtype=torch.int64, device=device if device is not None else "cuda")


class DecodeContext:
    """Device context of b64_decode_fused (B64_DECODE_CTX_BYTES): with it, decode_async is ONE
    kernel launch (no initialisation, no finalize launch).  Calls sharing a context must be
    ordered (one context per stream)."""

    def __init__(self, device=None, stream: Optional[torch.cuda.Stream] = None):
        self.buf = torch.empty(16, dtype=torch.uint8, device=device if device is not None else "cuda")
        _lib.check(_lib.lib().b64_decode_ctx_init(_ptr(self.buf), _stream(stream)), "b64_decode_ctx_init")


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
    if m % 4:
        raise B64Error("B64_ELENGTH: text length is not a multiple of 4")
    if out is None:
        out = torch.empty(max(decoded_len_max(m), 1), dtype=torch.uint8, device=t.device)
    if info is None:
        info = new_info(t.device)
    ip = info.data_ptr()
    if ctx is not None:
        _lib.check(_lib.lib().b64_decode_fused(_ptr(t), m, _ptr(out), _alpha(a), ctypes.c_void_p(ip),
                                               ctypes.c_void_p(ip + 8), ctypes.c_void_p(ip + 16), _ptr(ctx.buf),
                                               _stream(stream)), "b64_decode_fused")
        return out, info
    _lib.check(_lib.lib().b64_decode_ex(_ptr(t), m, _ptr(out), _alpha(a), ctypes.c_void_p(ip),
                                        ctypes.c_void_p(ip + 8), ctypes.c_void_p(ip + 16), _stream(stream)),
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
    err, _, olen = info.tolist()
    return out[:olen], err


def decode_unpadded(t: torch.Tensor, a: Optional[Alphabet] = None, out: Optional[torch.Tensor] = None,
                    stream: Optional[torch.cuda.Stream] = None) -> Tuple[torch.Tensor, int]:
    """Padding-optional validating decode (b64_decode_unpadded, R13).
    Returns (decoded bytes, err_off); err_off = -1 when valid."""
    _check_u8(t, "t")
    m = t.numel()
    if m % 4 == 1:
        raise B64Error("B64_ELENGTH: text length is 1 more than a multiple of 4")
    if out is None:
        out = torch.empty(3 * (m // 4) + 3, dtype=torch.uint8, device=t.device)
    info = new_info(t.device)
    ip = info.data_ptr()
    _lib.check(_lib.lib().b64_decode_unpadded(_ptr(t), m, _ptr(out), _alpha(a), ctypes.c_void_p(ip),
                                              ctypes.c_void_p(ip + 8), ctypes.c_void_p(ip + 16), _stream(stream)),
               "b64_decode_unpadded")
    err, _, olen = info.tolist()
    return out[:olen], err


def decode_ws(t: torch.Tensor, a: Optional[Alphabet] = None, out: Optional[torch.Tensor] = None,
              workspace: Optional[torch.Tensor] = None,
              stream: Optional[torch.cuda.Stream] = None) -> Tuple[torch.Tensor, int]:
    """Whitespace-skipping validating decode (b64_decode_ws, R14): MIME-style line
    breaks and blanks are ignored; err_off is a position in the ORIGINAL text (-1 = valid)."""
    _check_u8(t, "t")
    m = t.numel()
    if out is None:
        out = torch.empty(max(3 * (m // 4), 1), dtype=torch.uint8, device=t.device)
    need = int(_lib.lib().b64_decode_ws_workspace_bytes(m))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=t.device)
    info = new_info(t.device)
    ip = info.data_ptr()
    _lib.check(_lib.lib().b64_decode_ws(_ptr(t), m, _ptr(out), _alpha(a), _ptr(workspace), workspace.numel(),
                                        ctypes.c_void_p(ip), ctypes.c_void_p(ip + 8), ctypes.c_void_p(ip + 16),
                                        _stream(stream)), "b64_decode_ws")
    err, _, olen = info.tolist()
    return out[:olen], err


def decode_chunk(t: torch.Tensor, base_offset: int, is_final: bool, err_cell: torch.Tensor,
                 a: Optional[Alphabet] = None, out: Optional[torch.Tensor] = None,
                 out_len: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Shard-aware decode (b64_decode_chunk): lowers err_cell (int64[1], init ERR_NONE) with the
    packed first error (global_pos << 3 | status)."""
    _check_u8(t, "t")
    _check_i64(err_cell, "err_cell")
    m = t.numel()
    if out is None:
        out = torch.empty(max(decoded_len_max(m), 1), dtype=torch.uint8, device=t.device)
    _lib.check(_lib.lib().b64_decode_chunk(_ptr(t), m, _ptr(out), _alpha(a), base_offset, 1 if is_final else 0,
                                           _ptr(err_cell), _ptr(out_len), _stream(stream)), "b64_decode_chunk")
    return out


def decode_finalize(err_cell: torch.Tensor, err_off: torch.Tensor, status: Optional[torch.Tensor] = None,
                    stream: Optional[torch.cuda.Stream] = None) -> None:
    """Packed error word -> (err_off = -1 | position, status) on the device."""
    _check_i64(err_cell, "err_cell")
    _check_i64(err_off, "err_off")
    _lib.check(_lib.lib().b64_decode_finalize(_ptr(err_cell), _ptr(err_off), _ptr(status), _stream(stream)),
               "b64_decode_finalize")


# ------------------------------------------------------------------ grouped launches

def _enc_items(xs, alphabets, outs):
    k = len(xs)
    al = alphabets if isinstance(alphabets, (list, tuple)) else [alphabets] * k
    al = [a if a is not None else standard() for a in al]
    if outs is None:
        outs = [torch.empty(encoded_len(x.numel()), dtype=torch.uint8, device=x.device) for x in xs]
    items = (_lib.EncodeItem * max(k, 1))()
    for i, (x, o) in enumerate(zip(xs, outs)):
        _check_u8(x, "x")
        _check_u8(o, "out")
        items[i] = _lib.EncodeItem(x.data_ptr(), x.numel(), o.data_ptr(), ctypes.pointer(al[i]))
    return items, [o[: encoded_len(x.numel())] for x, o in zip(xs, outs)]


def _dec_items(ts, alphabets, outs, cells, bases, finals):
    k = len(ts)
    dev = ts[0].device
    al = alphabets if isinstance(alphabets, (list, tuple)) else [alphabets] * k
    al = [a if a is not None else standard() for a in al]
    if outs is None:
        outs = [torch.empty(max(decoded_len_max(t.numel()), 1), dtype=torch.uint8, device=dev) for t in ts]
    if cells is None:
        cells = torch.full((k,), ERR_NONE, dtype=torch.int64, device=dev)
    items = (_lib.DecodeItem * max(k, 1))()
    for i, (t, o) in enumerate(zip(ts, outs)):
        _check_u8(t, "t")
        if t.numel() % 4:
            raise B64Error("B64_ELENGTH: text length is not a multiple of 4")
        items[i] = _lib.DecodeItem(t.data_ptr(), t.numel(), o.data_ptr(), ctypes.pointer(al[i]),
                                   0 if bases is None else bases[i], 1 if finals is None else int(finals[i]), 0,
                                   cells[i:].data_ptr())
    return items, outs, cells


def _finalize_n(cells, k, dev, stream):
    err = torch.empty(k, dtype=torch.int64, device=dev)
    st = torch.empty(k, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().b64_decode_finalize_n(_ptr(cells), k, _ptr(err), _ptr(st), _stream(stream)),
               "b64_decode_finalize_n")
    return err, st


def encode_group(xs, alphabets=None, outs=None, stream: Optional[torch.cuda.Stream] = None):
    """Encode several independent device buffers with one kernel per group of 8 (b64_encode_group).
    alphabets: one Alphabet for all, or a list; returns the list of outputs."""
    items, outs = _enc_items(xs, alphabets, outs)
    _lib.check(_lib.lib().b64_encode_group(items, len(xs), _stream(stream)), "b64_encode_group")
    return outs


def decode_group(ts, alphabets=None, outs=None, cells: Optional[torch.Tensor] = None, bases=None, finals=None,
                 stream: Optional[torch.cuda.Stream] = None):
    """Validating decode of several device buffers, one kernel per group of 8 (b64_decode_group).
    Returns (outs, err_off int64[k] device tensor, status int32[k] device tensor)."""
    items, outs, cells = _dec_items(ts, alphabets, outs, cells, bases, finals)
    _lib.check(_lib.lib().b64_decode_group(items, len(ts), _stream(stream)), "b64_decode_group")
    err, st = _finalize_n(cells, len(ts), ts[0].device, stream)
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
    eitems, eouts = _enc_items(xs, enc_alphabets, enc_outs)
    if ts:
        ditems, douts, cells = _dec_items(ts, dec_alphabets, dec_outs, cells, None, None)
    else:
        ditems, douts = (_lib.DecodeItem * 1)(), []
    if ticket is None:
        ticket = torch.zeros(1, dtype=torch.int32, device=dev)
    k = max(len(ts), 1)
    err = err if err is not None else torch.empty(k, dtype=torch.int64, device=dev)
    status = status if status is not None else torch.empty(k, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().b64_codec_group_fused(eitems, len(xs), ditems, len(ts), _ptr(err), _ptr(status),
                                                _ptr(ticket), _stream(stream)), "b64_codec_group_fused")
    return eouts, douts, err[: len(ts)], status[: len(ts)]


def codec_group(xs, ts, enc_alphabets=None, dec_alphabets=None, enc_outs=None, dec_outs=None,
                cells: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None):
    """Independent encodes of xs and validating decodes of ts, ONE kernel per group of up to 8 + 8
    (b64_codec_group).  Returns (encoded list, decoded list, err_off int64[len(ts)] or None,
    status int32[len(ts)] or None)."""
    eitems, eouts = _enc_items(xs, enc_alphabets, enc_outs)
    if ts:
        ditems, douts, cells = _dec_items(ts, dec_alphabets, dec_outs, cells, None, None)
    else:
        ditems, douts = (_lib.DecodeItem * 1)(), []
    _lib.check(_lib.lib().b64_codec_group(eitems, len(xs), ditems, len(ts), _stream(stream)), "b64_codec_group")
    if not ts:
        return eouts, douts, None, None
    err, st = _finalize_n(cells, len(ts), ts[0].device, stream)
    return eouts, douts, err, st


# ------------------------------------------------------------------ streaming (carry between calls)

class EncodeStream:
    """Encode input that arrives in pieces of any length (b64_encode_stream_*).

    update(x) returns the chars completed so far (a view of a fresh or given buffer);
    end() returns the padded tail.  The concatenation of every returned piece equals
    encode(concatenation of the inputs)."""

    def __init__(self, a: Optional[Alphabet] = None, device=None, stream: Optional[torch.cuda.Stream] = None):
        self.a = _alpha(a)
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.carry = torch.zeros(8, dtype=torch.uint8, device=self.dev)
        self.st = _lib.Stream()
        self.stream = stream
        _lib.check(_lib.lib().b64_encode_stream_begin(ctypes.byref(self.st), _ptr(self.carry)),
                   "b64_encode_stream_begin")

    def out_len(self, n: int) -> int:
        return 4 * ((self.st.held + n) // 3)

    def update(self, x: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        _check_u8(x, "x")
        k = self.out_len(x.numel())
        if out is None:
            out = torch.empty(max(k, 1), dtype=torch.uint8, device=self.dev)
        n_out = ctypes.c_int64(0)
        _lib.check(_lib.lib().b64_encode_stream_update(ctypes.byref(self.st), _ptr(x), x.numel(), _ptr(out),
                                                       self.a, ctypes.byref(n_out), _stream(self.stream)),
                   "b64_encode_stream_update")
        return out[: n_out.value]

    def end(self, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        if out is None:
            out = torch.empty(4, dtype=torch.uint8, device=self.dev)
        n_out = ctypes.c_int64(0)
        _lib.check(_lib.lib().b64_encode_stream_end(ctypes.byref(self.st), _ptr(out), self.a, ctypes.byref(n_out),
                                                    _stream(self.stream)), "b64_encode_stream_end")
        return out[: n_out.value]


class DecodeStream:
    """Validating decode of text that arrives in pieces of any length (b64_decode_stream_*).

    update(t) returns the bytes of the quads completed so far (the last 1-4 chars are
    held back); end() returns (tail bytes tensor, info) with info = int64[3] device tensor
    (err_off, status, out_len) for the whole concatenated text, exactly as decode_async."""

    def __init__(self, a: Optional[Alphabet] = None, device=None, stream: Optional[torch.cuda.Stream] = None):
        self.a = _alpha(a)
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.carry = torch.zeros(8, dtype=torch.uint8, device=self.dev)
        self.cell = torch.empty(1, dtype=torch.int64, device=self.dev)
        self.st = _lib.Stream()
        self.stream = stream
        _lib.check(_lib.lib().b64_decode_stream_begin(ctypes.byref(self.st), _ptr(self.carry), _ptr(self.cell),
                                                      _stream(stream)), "b64_decode_stream_begin")

    def out_len(self, m: int) -> int:
        A = self.st.held + m
        return 3 * ((A - 1) // 4) if A > 0 else 0

    def update(self, t: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        _check_u8(t, "t")
        k = self.out_len(t.numel())
        if out is None:
            out = torch.empty(max(k, 1), dtype=torch.uint8, device=self.dev)
        n_out = ctypes.c_int64(0)
        _lib.check(_lib.lib().b64_decode_stream_update(ctypes.byref(self.st), _ptr(t), t.numel(), _ptr(out),
                                                       self.a, ctypes.byref(n_out), _stream(self.stream)),
                   "b64_decode_stream_update")
        return out[: n_out.value]

    def end(self, out: Optional[torch.Tensor] = None):
        if out is None:
            out = torch.empty(3, dtype=torch.uint8, device=self.dev)
        info = new_info(self.dev)
        ip = info.data_ptr()
        n_out = ctypes.c_int64(0)
        _lib.check(_lib.lib().b64_decode_stream_end(ctypes.byref(self.st), _ptr(out), self.a, ctypes.c_void_p(ip),
                                                    ctypes.c_void_p(ip + 8), ctypes.c_void_p(ip + 16),
                                                    ctypes.byref(n_out), _stream(self.stream)),
                   "b64_decode_stream_end")
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
        self.info = torch.zeros(2, dtype=torch.int64, device=dev)

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
            out = torch.empty(m, dtype=torch.uint8, pin_memory=True)
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
        """Returns (host bytes, err_off) when sync, else (host buffer, device info int64[2] = err, status;
        a fresh one per call unless `info` is given -- overlapped calls must not share it)."""
        if t.is_cuda or t.dtype != torch.uint8 or not t.is_contiguous():
            raise B64Error("t must be a contiguous uint8 host tensor (pinned for overlap)")
        m = t.numel()
        if m % 4:
            raise B64Error("B64_ELENGTH: text length is not a multiple of 4")
        if out is None:
            out = torch.empty(max(3 * (m // 4), 1), dtype=torch.uint8, pin_memory=True)
        if info is None:
            info = self.info if sync else torch.zeros(2, dtype=torch.int64, device=self.device)
        w = self._begin()
        with torch.cuda.stream(self.streams[1]):
            info[1].zero_()
        st = info[1:2].view(torch.int32)[:1]
        _lib.check(_lib.lib().b64_decode_host_ex(_ptr(t), m, _ptr(out), _alpha(a), _ptr(self.ws[w]), self.ws_bytes,
                                                 _ptr(info[0:1]), _ptr(st), *self._sp(), _lib.HOST_CALLER_ORDERED),
                   "b64_decode_host_ex")
        self._end(w)
        if not sync:
            return out, info
        self.join()
        err = int(info[0].item())
        if err < 0:
            pads = (2 if m >= 4 and int(t[m - 2]) == (a or standard()).pad else
                    (1 if m >= 4 and int(t[m - 1]) == (a or standard()).pad else 0))
            olen = 3 * (m // 4) - pads
        else:
            olen = 3 * (err // 4)
        return out[:olen], err


# ------------------------------------------------------------------ batched

def encode_batch(x: torch.Tensor, in_off: torch.Tensor, a: Optional[Alphabet] = None,
                 out: Optional[torch.Tensor] = None, out_off: Optional[torch.Tensor] = None,
                 total_out: Optional[int] = None,
                 stream: Optional[torch.cuda.Stream] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Per-string padded encode of strings concatenated in x (offsets int64[count+1]).
    Returns (out, out_off) with out_off = exclusive scan of 4*ceil(len/3) (int64[count+1])."""
    _check_u8(x, "x")
    if x.numel() == 0:  # all strings empty: the C ABI still wants a valid (unread) pointer
        x = torch.empty(1, dtype=torch.uint8, device=x.device)
    _check_i64(in_off, "in_off")
    count = in_off.numel() - 1
    if out_off is None:
        lens = in_off[1:] - in_off[:-1]
        out_off = torch.zeros(count + 1, dtype=torch.int64, device=x.device)
        torch.cumsum(4 * torch.div(lens + 2, 3, rounding_mode="floor"), 0, out=out_off[1:])
    if out is None:
        if total_out is None:
            total_out = int(out_off[-1].item())
        out = torch.empty(max(total_out, 1), dtype=torch.uint8, device=x.device)
    _lib.check(_lib.lib().b64_encode_batch(_ptr(x), _ptr(in_off), count, _ptr(out), _ptr(out_off), _alpha(a),
                                           _stream(stream)), "b64_encode_batch")
    return out, out_off


def decode_batch(t: torch.Tensor, in_off: torch.Tensor, a: Optional[Alphabet] = None,
                 out: Optional[torch.Tensor] = None, out_off: Optional[torch.Tensor] = None,
                 total_out: Optional[int] = None, stream: Optional[torch.cuda.Stream] = None,
                 index_base: int = 0, first_bad: Optional[torch.Tensor] = None):
    """Per-string validating decode.  Returns (out, out_off, status int32, err_off int64
    (relative, -1 = ok), out_len int64); out_off = exclusive scan of 3*(len//4).
    first_bad (device int64[1], caller-initialised, e.g. ERR_NONE): lowered to index_base + the
    index of the first failing string (b64_decode_batch_ex)."""
    _check_u8(t, "t")
    if t.numel() == 0:  # all strings empty: the C ABI still wants a valid (unread) pointer
        t = torch.empty(1, dtype=torch.uint8, device=t.device)
    _check_i64(in_off, "in_off")
    count = in_off.numel() - 1
    dev = t.device
    if out_off is None:
        lens = in_off[1:] - in_off[:-1]
        out_off = torch.zeros(count + 1, dtype=torch.int64, device=dev)
        torch.cumsum(3 * torch.div(lens, 4, rounding_mode="floor"), 0, out=out_off[1:])
    if out is None:
        if total_out is None:
            total_out = int(out_off[-1].item())
        out = torch.empty(max(total_out, 1), dtype=torch.uint8, device=dev)
    status = torch.empty(max(count, 1), dtype=torch.int32, device=dev)
    err = torch.empty(max(count, 1), dtype=torch.int64, device=dev)
    olen = torch.empty(max(count, 1), dtype=torch.int64, device=dev)
    if first_bad is not None:
        _check_i64(first_bad, "first_bad")
    _lib.check(_lib.lib().b64_decode_batch_ex(_ptr(t), _ptr(in_off), count, _ptr(out), _ptr(out_off), _alpha(a),
                                              _ptr(status), _ptr(err), _ptr(olen), index_base,
                                              _ptr(first_bad) if first_bad is not None else None, _stream(stream)),
               "b64_decode_batch_ex")
    return out, out_off, status[:count], err[:count], olen[:count]


def launch_count() -> int:
    """Kernels this process launched through the library (host-side counter)."""
    return int(_lib.lib().b64_launch_count())


def build_info() -> str:
    return _lib.lib().b64_build_info().decode()
