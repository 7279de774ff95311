"""The C-ABI library loads and exports every symbol include/b64gpu.h declares;
host-only logic (alphabet validation, sizes, synchronous argument errors) is
exercised without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "b64gpu.h")


@pytest.fixture(scope="module")
def L():
    import __graft_entry__ as g

    g.build()
    from paper_1910_05109_b200 import _lib

    return _lib.lib()


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(b64_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(L):
    names = header_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(L, n), n
    from paper_1910_05109_b200 import _lib

    assert sorted(s[0] for s in _lib.SIGNATURES) == names


def test_header_compiles_as_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "b64gpu.h"\nint main(void){ b64_alphabet a; return (int)sizeof(a) - 324; }\n')
    import subprocess

    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-c",
                           str(src), "-o", str(tmp_path / "t.o")])


def test_alphabet_host_logic(L):
    import paper_1910_05109_b200 as b64
    from paper_1910_05109_b200 import _lib

    std = b64.standard()
    assert bytes(std.enc) == b"ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/"
    assert bytes(b64.url().enc)[62:] == b"-_"
    assert std.pad == ord("=")
    dec = bytes(std.dec)
    assert sum(1 for v in dec if v != 0x80) == 64
    assert all(dec[c] == v for v, c in enumerate(std.enc))
    # Fig. 2: 'd' -> 0x1d, '6' -> 0x3a; 0xff and 0xc3 invalid
    assert dec[ord("d")] == 0x1D and dec[ord("6")] == 0x3A and dec[0xFF] == 0x80 and dec[0xC3] == 0x80
    with pytest.raises(_lib.B64Error, match="DUP"):
        b64.alphabet(b"A" * 64)
    with pytest.raises(_lib.B64Error, match="PAD"):
        b64.alphabet(bytes(std.enc), b"A")
    with pytest.raises(_lib.B64Error, match="NONASCII"):
        b64.alphabet(bytes(std.enc)[:63] + b"\xc3")
    a = b64.alphabet(bytes(reversed(bytes(std.enc))), b"!")
    assert a.dec[ord("/")] == 0 and a.pad == ord("!")


def test_sizes_and_sync_errors(L):
    assert L.b64_encoded_len(0) == 0 and L.b64_encoded_len(1) == 4 and L.b64_encoded_len(1048576) == 1398104
    assert L.b64_encoded_len(-1) == -1
    assert L.b64_decoded_len_max(1398104) == 1048578
    a = L.b64_alphabet_standard()
    # argument errors are synchronous and touch no device
    assert L.b64_encode(None, -1, None, a, None) == -1
    assert L.b64_encode(None, 0, None, a, None) == 0  # empty input: nothing launched
    assert L.b64_encode(None, 5, None, a, None) == -1
    assert L.b64_decode(None, 5, None, a, ctypes.c_void_p(8), None) == -2  # m % 4 != 0
    assert L.b64_decode(None, 4, None, a, None, None) == -1
    assert L.b64_decode_chunk(None, 6, None, a, 0, 1, ctypes.c_void_p(8), None, None) == -2
    assert L.b64_encode_batch(None, None, -1, None, None, a, None) == -1
    assert L.b64_encode_batch(None, None, 0, None, None, a, None) == 0
    # b64_decode_batch_ex: negative index base, index overflow with a first-bad word
    V = ctypes.c_void_p
    assert L.b64_decode_batch_ex(V(8), V(8), 1, V(8), V(8), a, None, V(8), None, -1, None, None) == -1
    assert L.b64_decode_batch_ex(V(8), V(8), 2, V(8), V(8), a, None, V(8), None, (1 << 63) - 1, V(8), None) == -1
    assert L.b64_decode_batch_ex(None, None, 0, None, None, a, None, None, None, 0, V(8), None) == 0
    # fused peer codec: world / rank out of range (nothing launched)
    assert L.b64_codec_group_fused_peer(None, 0, None, 0, V(8), None, V(8), V(8), 33, 0, 0, None) == -1
    assert L.b64_codec_group_fused_peer(None, 0, None, 0, V(8), None, V(8), V(8), 2, 2, 0, None) == -1
    assert L.b64_peer_combine_bytes(-1) == -1 and L.b64_peer_combine_bytes(0) == 64
    assert L.b64_peer_combine_bytes(6) == 2 * 32 * 6 * 16
    assert b"sm_100a" in L.b64_build_info()


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle and has no CPU codec path."""
    pkg = os.path.join(ROOT, "paper_1910_05109_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                s = open(os.path.join(dp, f)).read()
                assert "oracle" not in s.replace("oracle/", ""), f


def test_stream_host_state_machine(L):
    """Streaming API (b64gpu.h, R15): argument / state errors are synchronous
    and touch no device; zero-length pieces launch nothing."""
    from paper_1910_05109_b200 import _lib

    a = L.b64_alphabet_standard()
    st = _lib.Stream()
    n_out = ctypes.c_int64(-1)
    carry = ctypes.c_void_p(0x1000)  # never dereferenced on the host
    assert L.b64_encode_stream_update(ctypes.byref(st), None, 0, None, a, ctypes.byref(n_out), None) == -1  # not begun
    assert L.b64_encode_stream_begin(None, carry) == -1
    assert L.b64_encode_stream_begin(ctypes.byref(st), None) == -1
    assert L.b64_encode_stream_begin(ctypes.byref(st), carry) == 0
    assert (st.consumed, st.produced, st.held) == (0, 0, 0)
    assert L.b64_encode_stream_update(ctypes.byref(st), None, 0, None, a, ctypes.byref(n_out), None) == 0
    assert n_out.value == 0
    assert L.b64_encode_stream_update(ctypes.byref(st), None, 5, None, a, ctypes.byref(n_out), None) == -1
    assert L.b64_encode_stream_update(ctypes.byref(st), None, -1, None, a, ctypes.byref(n_out), None) == -1
    # a decode call on an encode stream is refused
    assert L.b64_decode_stream_update(ctypes.byref(st), None, 0, None, a, ctypes.byref(n_out), None) == -1
    assert L.b64_decode_stream_end(ctypes.byref(st), None, a, ctypes.c_void_p(8), None, None, None, None) == -1
    # nothing held: ending writes nothing and launches nothing
    assert L.b64_encode_stream_end(ctypes.byref(st), None, a, ctypes.byref(n_out), None) == 0
    assert n_out.value == 0
    assert L.b64_encode_stream_update(ctypes.byref(st), None, 0, None, a, ctypes.byref(n_out), None) == -1  # finished
    assert L.b64_decode_stream_begin(ctypes.byref(st), carry, None, None) == -1
