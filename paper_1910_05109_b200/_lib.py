"""ctypes loader for libb64gpu.so (the C ABI of include/b64gpu.h).

Argument marshalling only.  There is deliberately no fallback: if the shared
library is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libb64gpu.so")

B64_OK = 0
B64_EINVAL = -1
B64_ELENGTH = -2
B64_EALPHA_DUP = -3
B64_EALPHA_NONASCII = -4
B64_EALPHA_PAD = -5
B64_ECUDA = -6

ERR_NONE = 0x7F7F7F7F7F7F7F7F

ST_OK, ST_BADCHAR, ST_BADPAD, ST_NONCANON, ST_LENGTH = 0, 1, 2, 3, 4

ERRORS = {
    B64_EINVAL: "B64_EINVAL",
    B64_ELENGTH: "B64_ELENGTH",
    B64_EALPHA_DUP: "B64_EALPHA_DUP",
    B64_EALPHA_NONASCII: "B64_EALPHA_NONASCII",
    B64_EALPHA_PAD: "B64_EALPHA_PAD",
    B64_ECUDA: "B64_ECUDA",
}

# (name, restype, argtypes) for every symbol include/b64gpu.h declares.
P, I64, I32, INT = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int


ALPHA_LENIENT = 1  # B64_ALPHA_LENIENT
DECODE_CTX_BYTES = 16  # B64_DECODE_CTX_BYTES
BATCH_CTX_BYTES = 32  # B64_BATCH_CTX_BYTES
HOST_CALLER_ORDERED = 1  # B64_HOST_CALLER_ORDERED


class Alphabet(ctypes.Structure):
    _fields_ = [("enc", ctypes.c_uint8 * 64), ("dec", ctypes.c_uint8 * 256), ("pad", ctypes.c_uint8),
                ("flags", ctypes.c_uint8), ("reserved", ctypes.c_uint8 * 2)]


AP = ctypes.POINTER(Alphabet)


class EncodeItem(ctypes.Structure):
    _fields_ = [("d_in", ctypes.c_void_p), ("n", ctypes.c_int64), ("d_out", ctypes.c_void_p), ("a", AP)]


class DecodeItem(ctypes.Structure):
    _fields_ = [("d_in", ctypes.c_void_p), ("m", ctypes.c_int64), ("d_out", ctypes.c_void_p), ("a", AP),
                ("base_offset", ctypes.c_int64), ("is_final", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("d_err_min", ctypes.c_void_p)]

class Stream(ctypes.Structure):
    """b64_stream (streaming encode / decode state; lengths only, the carry is on the device)."""
    _fields_ = [("consumed", ctypes.c_int64), ("produced", ctypes.c_int64), ("held", ctypes.c_int32),
                ("state", ctypes.c_int32), ("d_carry", ctypes.c_void_p), ("d_err_min", ctypes.c_void_p)]


class Shard(ctypes.Structure):
    """b64_shard (multi-GPU sharding rule, host only)."""
    _fields_ = [("start", ctypes.c_int64), ("stop", ctypes.c_int64), ("out_start", ctypes.c_int64),
                ("out_len", ctypes.c_int64), ("is_final", ctypes.c_int32), ("reserved", ctypes.c_int32)]


SP = ctypes.POINTER(Stream)
STREAM_OVERLAP = 1  # B64_STREAM_OVERLAP
# b64_consumer_fn: (const uint8_t* d_chunk, int64 len, int64 out_offset, void* user, stream)
CONSUMER_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p)
I64P = ctypes.POINTER(ctypes.c_int64)

SIGNATURES = [
    ("b64_alphabet_init", INT, [AP, ctypes.c_char_p, ctypes.c_char, ctypes.POINTER(INT)]),
    ("b64_alphabet_set_flags", INT, [AP, ctypes.c_uint]),
    ("b64_alphabet_standard", AP, []),
    ("b64_alphabet_url", AP, []),
    ("b64_encoded_len", I64, [I64]),
    ("b64_decoded_len_max", I64, [I64]),
    ("b64_decoded_len_max_unpadded", I64, [I64]),
    ("b64_encode", INT, [P, I64, P, AP, P]),
    ("b64_decode", INT, [P, I64, P, AP, P, P]),
    ("b64_decode_ex", INT, [P, I64, P, AP, P, P, P, P]),
    ("b64_decode_unpadded", INT, [P, I64, P, AP, P, P, P, P]),
    ("b64_decode_ws_workspace_bytes", I64, [I64]),
    ("b64_decode_ws", INT, [P, I64, P, AP, P, I64, P, P, P, P]),
    ("b64_decode_chunk", INT, [P, I64, P, AP, I64, INT, P, P, P]),
    ("b64_decode_finalize", INT, [P, P, P, P]),
    ("b64_encode_shard", INT, [I64, INT, INT, ctypes.POINTER(Shard)]),
    ("b64_decode_shard", INT, [I64, INT, INT, ctypes.POINTER(Shard)]),
    ("b64_encode_group", INT, [P, I64, P]),
    ("b64_decode_group", INT, [P, I64, P]),
    ("b64_codec_group", INT, [P, I64, P, I64, P]),
    ("b64_codec_group_fused", INT, [P, I64, P, I64, P, P, P, P]),
    ("b64_codec_group_fused_peer", INT, [P, I64, P, I64, P, P, P, P, INT, INT, ctypes.c_uint64, P]),
    ("b64_decode_finalize_n", INT, [P, I64, P, P, P]),
    ("b64_stream_update_len", I64, [SP, I64]),
    ("b64_stream_end_len", I64, [SP]),
    ("b64_encode_stream_begin", INT, [SP, P]),
    ("b64_encode_stream_begin_ex", INT, [SP, P, ctypes.c_uint32, P]),
    ("b64_encode_stream_update", INT, [SP, P, I64, P, AP, I64P, P]),
    ("b64_encode_stream_end", INT, [SP, P, AP, I64P, P]),
    ("b64_decode_stream_begin", INT, [SP, P, P, P]),
    ("b64_decode_stream_begin_ex", INT, [SP, P, P, ctypes.c_uint32, P]),
    ("b64_decode_stream_update", INT, [SP, P, I64, P, AP, I64P, P]),
    ("b64_decode_stream_end", INT, [SP, P, AP, P, P, P, I64P, P]),
    ("b64_peer_combine_bytes", I64, [I64]),
    ("b64_peer_combine_init", INT, [P, I64, P]),
    ("b64_peer_combine", INT, [P, INT, INT, P, I64, ctypes.c_uint64, P, P, P]),
    ("b64_peer_buffer_alloc", INT, [I64, ctypes.POINTER(ctypes.c_void_p), ctypes.c_char_p]),
    ("b64_peer_buffer_open", INT, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    ("b64_peer_buffer_release", INT, [P, INT]),
    ("b64_peer_combine_emulate", INT, [P, INT, P, I64, INT, P, P, P]),
    ("b64_host_workspace_bytes", I64, [I64]),
    ("b64_encode_host", INT, [P, I64, P, AP, P, I64, P, P, P]),
    ("b64_decode_host", INT, [P, I64, P, AP, P, I64, P, P, P, P, P, P]),
    ("b64_encode_host_ex", INT, [P, I64, P, AP, P, I64, P, P, P, ctypes.c_uint]),
    ("b64_decode_host_ex", INT, [P, I64, P, AP, P, I64, P, P, P, P, P, P, ctypes.c_uint]),
    ("b64_encode_batch_offsets", INT, [P, I64, P, P]),
    ("b64_consume_chunk_chars", I64, [I64]),
    ("b64_decode_consume", INT, [P, I64, P, I64, AP, CONSUMER_FN, P, P, P, P, P]),
    ("b64_decode_batch_offsets", INT, [P, I64, P, P]),
    ("b64_encode_batch", INT, [P, P, I64, P, P, AP, P]),
    ("b64_decode_batch", INT, [P, P, I64, P, P, AP, P, P, P, P]),
    ("b64_decode_batch_ex", INT, [P, P, I64, P, P, AP, P, P, P, I64, P, P]),
    ("b64_decode_ctx_init", INT, [P, P]),
    ("b64_batch_ctx_init", INT, [P, P]),
    ("b64_decode_batch_fast", INT, [P, P, I64, P, P, AP, P, P, P, I64, P, P, P]),
    ("b64_decode_fused", INT, [P, I64, P, AP, P, P, P, P, P]),
    ("b64_launch_count", I64, []),
    ("b64_build_info", ctypes.c_char_p, []),
]

_lib = None


class B64Error(RuntimeError):
    pass


def lib():
    """Load the CUDA library (raises if it is missing: no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise B64Error(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc != B64_OK:
        raise B64Error(f"{what} failed: {ERRORS.get(rc, rc)}")
