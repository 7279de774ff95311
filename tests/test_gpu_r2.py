"""GPU parity, round 2: the brute-force domains through the CUDA kernels, the device-side
batch offsets, the closed boundary (exact lengths from the device, size queries), and the
stream / device / buffer discipline of the Python binding.

Every expected value comes from the oracle (oracle/) on the same inputs; the inputs are
enumerations (all triples, all quads, all padded final quads) or seeded synthetic data.
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def b64():
    import __graft_entry__ as g

    g.build()
    import paper_1910_05109_b200 as m

    assert torch.cuda.is_available()
    return m


def _alpha(b64, chars):
    return b64.standard() if chars == oracle.STANDARD else b64.url()


# ------------------------------------------------------------------ brute-force domains

def test_all_triples_encode(b64):
    """Every one of the 2^24 byte triples, as one 48 MiB stream: the fast
    kernel (aligned) and the generic kernel (input at +1, output at +3), both alphabets."""
    i = np.arange(1 << 24, dtype=np.uint32)
    x = np.stack([(i >> 16) & 0xFF, (i >> 8) & 0xFF, i & 0xFF], axis=1).astype(np.uint8).reshape(-1)
    for chars in (oracle.STANDARD, oracle.URL):
        ref = oracle.encode(x, chars)
        a = _alpha(b64, chars)
        xd = torch.from_numpy(x).to(DEV)
        got = b64.encode(xd, a)
        assert np.array_equal(got.cpu().numpy(), ref)
        buf = torch.empty(x.size + 1, dtype=torch.uint8, device=DEV)
        buf[1:] = xd
        ob = torch.empty(ref.size + 3, dtype=torch.uint8, device=DEV)
        b64.encode(buf[1:], a, out=ob[3:])
        assert np.array_equal(ob[3:].cpu().numpy(), ref)
        del xd, buf, ob, got
    torch.cuda.empty_cache()


def test_all_quads_decode(b64):
    """Every one of the 64^4 valid quads, as one 64 MiB text: bytes against
    the oracle, both alphabets, fast and generic kernels; then one non-alphabet byte at the
    very end of the enumeration (its final quad) and one in the middle."""
    i = np.arange(1 << 24, dtype=np.uint32)
    for chars in (oracle.STANDARD, oracle.URL):
        A = np.frombuffer(chars, np.uint8)
        t = np.stack([A[(i >> 18) & 63], A[(i >> 12) & 63], A[(i >> 6) & 63], A[i & 63]], axis=1).reshape(-1)
        ref, rerr, rst = oracle.decode(t, chars)
        assert rerr == -1 and ref.size == 3 << 24
        a = _alpha(b64, chars)
        td = torch.from_numpy(t).to(DEV)
        y, err = b64.decode(td, a)
        assert err == -1 and np.array_equal(y.cpu().numpy(), ref)
        buf = torch.empty(t.size + 5, dtype=torch.uint8, device=DEV)
        buf[5:] = td
        y, err = b64.decode(buf[5:], a)  # generic kernel
        assert err == -1 and np.array_equal(y.cpu().numpy(), ref)
        for p in (t.size // 2 + 1, t.size - 3):
            t2 = t.copy()
            t2[p] = ord("*")
            r2, e2, s2 = oracle.decode(t2, chars)
            y, info = b64.decode_async(torch.from_numpy(t2).to(DEV), a)
            err, st, olen = info.tolist()
            assert (err, st, olen) == (e2, s2, 3 * (e2 // 4)) and e2 == p
            assert np.array_equal(y[:olen].cpu().numpy(), r2)
        del td, buf
    torch.cuda.empty_cache()


@pytest.mark.parametrize("lenient", [False, True])
def test_all_padded_final_quads_batch(b64, lenient):
    """All 4,096 'xx==' and all 262,144 'xxx=' quads as a batch of
    4-char strings, strict and lenient (R6 / R16): status, err_off, out_len and bytes
    against the oracle; strict accepts exactly 256 + 65,536 of them."""
    A = np.frombuffer(oracle.STANDARD, np.uint8)
    p = ord("=")
    i2 = np.arange(64 * 64)
    q2 = np.stack([A[i2 >> 6], A[i2 & 63], np.full_like(i2, p), np.full_like(i2, p)], axis=1).astype(np.uint8)
    i3 = np.arange(64 ** 3)
    q3 = np.stack([A[i3 >> 12], A[(i3 >> 6) & 63], A[i3 & 63], np.full_like(i3, p)], axis=1).astype(np.uint8)
    t = np.concatenate([q2, q3]).reshape(-1)
    count = t.size // 4
    off = np.arange(count + 1, dtype=np.int64) * 4
    rout, roff, rst, rerr, rlen = oracle.decode_batch(t, off, lenient=lenient)
    a = b64.standard() if not lenient else b64.lenient_of(b64.standard())
    out, oo, st, err, olen = b64.decode_batch(torch.from_numpy(t).to(DEV), torch.from_numpy(off).to(DEV), a)
    assert np.array_equal(oo.cpu().numpy(), roff)
    assert np.array_equal(st.cpu().numpy(), rst)
    assert np.array_equal(err.cpu().numpy(), rerr)
    assert np.array_equal(olen.cpu().numpy(), rlen)
    if not lenient:
        assert int((rst == 0).sum()) == 256 + 65536
    else:
        assert int((rst == 0).sum()) == count
    o = out.cpu().numpy()
    for k in np.nonzero(rst == 0)[0][::97]:
        assert np.array_equal(o[roff[k]: roff[k] + rlen[k]], rout[roff[k]: roff[k] + rlen[k]])
    ok = np.nonzero(rst == 0)[0]
    # every accepted string's bytes: gather the first byte (always present) and compare in bulk
    assert np.array_equal(o[roff[ok]], rout[roff[ok]])
    two = ok[rlen[ok] >= 2]
    assert np.array_equal(o[roff[two] + 1], rout[roff[two] + 1])


def test_config3_encode_full_length(b64):
    """configs[2]'s 1 GiB encode (enc_fast_kernel<2>) compared over its whole 1.43 GB output,
    in 96 MiB windows cut at 3-byte boundaries (each window is the oracle's encode of its
    bytes; the last one carries the '==' padding)."""
    n = 1 << 30
    xd = synth.device_data(n, seed=0)
    t = b64.encode(xd)
    assert t.numel() == 1431655768
    W = 96 << 20  # a multiple of 3
    for s in range(0, n, W):
        e = min(n, s + W)
        ref = oracle.encode(xd[s:e].cpu().numpy())
        got = t[4 * (s // 3): 4 * (s // 3) + ref.size].cpu().numpy()
        assert np.array_equal(got, ref), s
    del xd, t
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ device-side batch offsets

@pytest.mark.parametrize("count", [0, 1, 2, 2047, 2048, 2049, 4096, 100_003])
def test_batch_offsets_vs_oracle(b64, count):
    """b64_encode_batch_offsets / b64_decode_batch_offsets (three-kernel device scan) against the
    oracle's offsets (exclusive scans of the length law / decode capacity); lengths include 0
    and every residue mod 3 and 4, offsets start at a non-zero base."""
    rng = np.random.default_rng(count)
    lens = rng.integers(0, 70, size=count).astype(np.int64)
    lens[::17] = 0
    off = np.concatenate([[13], 13 + np.cumsum(lens)]).astype(np.int64)
    d = torch.from_numpy(off).to(DEV)
    x = synth.data(int(off[-1]) + 1, seed=count)
    _, eref = oracle.encode_batch(x, off)
    _, dref, *_ = oracle.decode_batch(x, off)
    assert np.array_equal(b64.encode_batch_offsets(d).cpu().numpy(), eref)
    assert np.array_equal(b64.decode_batch_offsets(d).cpu().numpy(), dref)


# ------------------------------------------------------------------ the closed boundary

def test_host_pipeline_length_from_device(b64):
    """HostPipeline.decode takes the exact output length from the device (b64_decode_host's
    d_out_len): valid texts with 0 / 1 / 2 pads, an error in the last chunk, an empty text."""
    pipe = b64.HostPipeline(chunk_bytes=3072 * 3)
    for n in (0, 1, 2, 3, 9216, 9217, 9218, 50_000):
        x = synth.data(n, seed=n)
        ref = oracle.encode(x)
        y, err = pipe.decode(torch.from_numpy(ref.copy()).pin_memory())
        assert err == -1 and y.numel() == n and np.array_equal(y.numpy(), x)
        if ref.size >= 8:
            t2 = ref.copy()
            t2[-6] = ord("#")
            rr, re, rs = oracle.decode(t2)
            yo, info = pipe.decode(torch.from_numpy(t2).pin_memory(), sync=False)
            pipe.join()
            torch.cuda.synchronize()
            err, _, olen = info.tolist()
            assert (err, olen) == (re, rr.size) and np.array_equal(yo[:olen].numpy(), rr)


def test_unpadded_and_stream_sizes_from_library(b64):
    """decode_unpadded's buffer and the stream pieces' sizes come from the library's queries;
    results against the oracle for every tail length."""
    for n in range(0, 40):
        x = synth.data(n, seed=n + 3)
        tu = oracle.encode_unpadded(x, oracle.URL)
        y, err = b64.decode_unpadded(torch.from_numpy(tu.copy()).to(DEV), b64.url())
        assert err == -1 and np.array_equal(y.cpu().numpy(), x), n
    x = synth.data(10_007, seed=1)
    ref = oracle.encode(x)
    es = b64.EncodeStream()
    parts = [es.update(torch.from_numpy(x[a:b].copy()).to(DEV)) for a, b in ((0, 1), (1, 5), (5, 10_000), (10_000, 10_007))]
    parts.append(es.end())
    assert np.array_equal(torch.cat(parts).cpu().numpy(), ref)
    ds = b64.DecodeStream()
    cuts = (0, 3, 4, 7, 5000, ref.size)
    parts = [ds.update(torch.from_numpy(ref[a:b].copy()).to(DEV)) for a, b in zip(cuts, cuts[1:])]
    tail, info = ds.end()
    torch.cuda.synchronize()
    err, _, olen = info.tolist()
    got = torch.cat(parts + [tail]).cpu().numpy()
    assert err == -1 and np.array_equal(got[: x.size], x)


# ------------------------------------------------------------------ binding discipline

def test_explicit_stream_not_current(b64):
    """stream= a side stream while the current stream is busy: the wrappers order their scratch
    fills (info, cells, ticket) before the kernels and join before reading results
    (stream-ordering race)."""
    side = torch.cuda.Stream()
    x = synth.data(3 * 1024 * 1024 + 1, seed=5)
    ref = oracle.encode(x)
    t2 = ref.copy()
    t2[777] = ord("*")
    xd = torch.from_numpy(x).to(DEV)
    td = torch.from_numpy(t2).to(DEV)
    for rep in range(3):
        torch.cuda._sleep(20_000_000)  # the current stream stays busy for a while
        y, err = b64.decode(td, stream=side)
        assert err == 777
        torch.cuda._sleep(20_000_000)
        y, err = b64.decode_unpadded(td, stream=side)
        assert err == 777
        torch.cuda._sleep(20_000_000)
        outs, err, st = b64.decode_group([td, torch.from_numpy(ref).to(DEV)], stream=side)
        side.synchronize()
        assert err.tolist() == [777, -1]
        torch.cuda._sleep(20_000_000)
        eo, do, err, st = b64.codec_group_fused([xd], [td], stream=side)
        side.synchronize()
        assert err.tolist() == [777] and np.array_equal(eo[0].cpu().numpy(), ref)
    torch.cuda.synchronize()


def test_out_buffers_checked(b64):
    """Caller-supplied outputs are checked before any launch: too small, wrong dtype,
    host memory, wrong device -> B64Error, nothing launched."""
    x = torch.from_numpy(synth.data(3000, seed=2)).to(DEV)
    t = b64.encode(x)
    before = b64.launch_count()
    bad = [torch.empty(10, dtype=torch.uint8, device=DEV), torch.empty(t.numel(), dtype=torch.int16, device=DEV),
           torch.empty(t.numel(), dtype=torch.uint8)]
    for o in bad:
        with pytest.raises(b64.B64Error):
            b64.encode(x, out=o)
        with pytest.raises(b64.B64Error):
            b64.decode_async(t, out=o)
        with pytest.raises(b64.B64Error):
            b64.decode_chunk(t, 0, True, torch.full((1,), b64.ERR_NONE, dtype=torch.int64, device=DEV), out=o)
    with pytest.raises(b64.B64Error):
        b64.decode_ws(t, out=torch.empty(5, dtype=torch.uint8, device=DEV))
    with pytest.raises(b64.B64Error):
        b64.encode_batch(x, torch.tensor([0, 3000], dtype=torch.int64, device=DEV),
                         out=torch.empty(5, dtype=torch.uint8, device=DEV),
                         out_off=torch.tensor([0, 4000], dtype=torch.int64, device=DEV))
    es = b64.EncodeStream()
    with pytest.raises(b64.B64Error):
        es.update(x, out=torch.empty(1, dtype=torch.uint8, device=DEV))
    assert b64.launch_count() == before


# ------------------------------------------------------------------ batched decode: concatenation path

def _batch_case(count, seed, hi=3000):
    Ls = synth.loguniform_lengths(count, hi=hi, seed=seed)
    off = synth.offsets(Ls)
    x = synth.data(int(off[-1]), seed=seed)
    text, toff = oracle.encode_batch(x, off)
    return text, toff


@pytest.mark.parametrize("lenient", [False, True])
def test_batch_fast_path_vs_oracle(b64, lenient):
    """b64_decode_batch_fast: eligible batches (every length a
    multiple of 4) with corruptions of every kind -- non-alphabet bytes, '=' in the middle of a
    string (the pad-count mismatch -> per-string fallback), '=' at len-3, data after '=',
    non-canonical final quads -- against the oracle, strict and lenient; and the same batch
    through the generic path (fast=False) gives identical results."""
    a = b64.standard() if not lenient else b64.lenient_of(b64.standard())
    text, toff = _batch_case(4000, seed=21)
    count = toff.size - 1
    rng = np.random.default_rng(21)
    variants = {"clean": text.copy()}
    t = text.copy()
    for s in rng.choice(count, 40, replace=False):  # non-alphabet bytes anywhere
        L = toff[s + 1] - toff[s]
        t[toff[s] + rng.integers(0, L)] = ord("*")
    variants["badchar"] = t
    t = text.copy()
    for s in rng.choice(count, 7, replace=False):  # '=' inside a string: misplaced pad
        L = toff[s + 1] - toff[s]
        if L >= 8:
            t[toff[s] + rng.integers(0, L - 4)] = ord("=")
    variants["pad_inside"] = t
    t = text.copy()
    for s in rng.choice(count, 60, replace=False):  # final-quad forms: x=yy, xx=y, non-canonical
        e = toff[s + 1]
        k = int(rng.integers(0, 3))
        if k == 0:
            t[e - 3] = ord("=")
        elif k == 1:
            t[e - 2] = ord("=")
        else:
            t[e - 2], t[e - 1] = ord("B"), ord("=")  # 'xxB=': non-canonical (B = 1)
    variants["final_forms"] = t
    toff_d = torch.from_numpy(toff).to(DEV)
    for name, tv in variants.items():
        rout, roff, rst, rerr, rlen = oracle.decode_batch(tv, toff, lenient=lenient)
        td = torch.from_numpy(tv).to(DEV)
        res = {}
        for fast in (True, False):
            out, oo, st, err, olen = b64.decode_batch(td, toff_d, a, fast=fast)
            res[fast] = (st.cpu().numpy(), err.cpu().numpy(), olen.cpu().numpy(), out.cpu().numpy())
            assert np.array_equal(res[fast][0], rst), (name, fast)
            assert np.array_equal(res[fast][1], rerr), (name, fast)
            assert np.array_equal(res[fast][2], rlen), (name, fast)
            o = res[fast][3]
            ok = np.nonzero(rlen > 0)[0]
            for s in ok[::13]:
                assert np.array_equal(o[roff[s]: roff[s] + rlen[s]], rout[roff[s]: roff[s] + rlen[s]]), (name, s)
            # every string's exact bytes, gathered: the first and the last exact byte
            assert np.array_equal(o[roff[ok]], rout[roff[ok]]), name
            assert np.array_equal(o[roff[ok] + rlen[ok] - 1], rout[roff[ok] + rlen[ok] - 1]), name


def test_batch_fast_path_ineligible_layouts(b64):
    """Layouts the concatenation path must refuse (the per-string kernel runs): a length not a
    multiple of 4, a gap in the output offsets, a misaligned first string; empty strings and a
    batch of only empty strings; repeated calls reuse the cached context."""
    text, toff = _batch_case(3000, seed=22)
    cases = []
    t2 = np.concatenate([text[: toff[100]], np.frombuffer(b"QUJD", np.uint8)[:3], text[toff[100]:]])
    o2 = np.concatenate([toff[:101], toff[100:] + 3])
    cases.append(("len%4", t2, o2, None))
    _, doff, *_ = oracle.decode_batch(text, toff)
    gap = doff.copy()
    gap[1500:] += 16
    cases.append(("gap", text, toff, gap))
    t3 = np.concatenate([np.zeros(4, np.uint8), text])
    cases.append(("misaligned", t3, toff + 4, None))
    Lz = np.diff(toff).copy()
    Lz[::5] = 0
    tz = np.concatenate([text[toff[i]: toff[i] + Lz[i]] for i in range(Lz.size)])
    cases.append(("empties", tz, synth.offsets(Lz), None))
    cases.append(("all_empty", np.zeros(0, np.uint8), np.zeros(11, np.int64), None))
    for name, tv, off, oo in cases:
        rout, roff, rst, rerr, rlen = oracle.decode_batch(tv, off)
        for rep in range(2):
            kw = {}
            if oo is not None:
                kw = dict(out_off=torch.from_numpy(oo).to(DEV), total_out=int(oo[-1]) + 64)
            out, ooo, st, err, olen = b64.decode_batch(torch.from_numpy(tv).to(DEV), torch.from_numpy(off).to(DEV), **kw)
            assert np.array_equal(st.cpu().numpy(), rst), name
            assert np.array_equal(err.cpu().numpy(), rerr), name
            assert np.array_equal(olen.cpu().numpy(), rlen), name
            o = out.cpu().numpy()
            base = oo if oo is not None else roff
            for s in np.nonzero(rlen > 0)[0][::29]:
                assert np.array_equal(o[base[s]: base[s] + rlen[s]], rout[roff[s]: roff[s] + rlen[s]]), (name, s)


# ------------------------------------------------------------------ misaligned bulk decode (unaligned.cu)

@pytest.mark.parametrize("ioff", [1, 2, 3, 4, 5, 13, 31])
def test_decode_misaligned_fast_kernel(b64, ioff):
    """dec_fastu_kernel (any alignment, inputs of >= 64 Ki chars): every input offset mod 4 and
    several mod 32, output offsets mod 8, lengths with head / tail / final quads, valid and
    with a non-alphabet byte in the head, the bulk, the tail and the final quad -- against the
    oracle, exact bytes and out_len."""
    rng = np.random.default_rng(ioff)
    for n in (49_152 + 7, 200_003, 1_000_000):
        x = synth.data(n, seed=n + ioff)
        ref = oracle.encode(x)
        m = ref.size
        for ooff in (0, 1, 3, 5, 8):
            buf = torch.empty(m + 64, dtype=torch.uint8, device=DEV)
            tin = buf[ioff: ioff + m]
            tin.copy_(torch.from_numpy(ref).to(DEV))
            obuf = torch.empty(3 * (m // 4) + 64, dtype=torch.uint8, device=DEV)
            out = obuf[ooff: ooff + 3 * (m // 4)]
            y, info = b64.decode_async(tin, out=out)
            err, st, olen = info.tolist()
            assert err == -1 and olen == n and np.array_equal(y[:n].cpu().numpy(), x), (n, ooff)
        for p in (1, 9, 30, m // 2 + 3, m - 700, m - 6, m - 1):
            t2 = ref.copy()
            t2[p] = ord("!") if rng.random() < 0.5 else 0xC3
            r2, e2, s2 = oracle.decode(t2)
            buf = torch.empty(m + 64, dtype=torch.uint8, device=DEV)
            tin = buf[ioff: ioff + m]
            tin.copy_(torch.from_numpy(t2).to(DEV))
            obuf = torch.empty(3 * (m // 4) + 64, dtype=torch.uint8, device=DEV)
            out = obuf[3: 3 + 3 * (m // 4)]
            y, info = b64.decode_async(tin, out=out)
            err, st, olen = info.tolist()
            assert (err, st, olen) == (e2, s2, r2.size), (n, p)
            assert np.array_equal(y[:olen].cpu().numpy(), r2), (n, p)


def test_decode_misaligned_no_stray_writes(b64):
    """dec_fastu_kernel writes exactly [out, out + out_len): canary bytes before and after the
    output (and every byte of the partial 8-byte words at chunk edges) stay intact."""
    for n in (300_001, 1 << 20):
        x = synth.data(n, seed=n)
        ref = oracle.encode(x)
        m = ref.size
        for ioff, ooff in ((1, 1), (2, 7), (3, 4), (6, 3)):
            tb = torch.empty(m + 32, dtype=torch.uint8, device=DEV)
            tb[ioff: ioff + m] = torch.from_numpy(ref).to(DEV)
            ob = torch.full((3 * (m // 4) + 2 * 256,), 0xA5, dtype=torch.uint8, device=DEV)
            out = ob[256 + ooff: 256 + ooff + 3 * (m // 4)]
            y, info = b64.decode_async(tb[ioff: ioff + m], out=out)
            err, st, olen = info.tolist()
            assert err == -1 and olen == n
            h = ob.cpu().numpy()
            assert (h[: 256 + ooff] == 0xA5).all() and (h[256 + ooff + n:] == 0xA5).all(), (n, ioff, ooff)
            assert np.array_equal(h[256 + ooff: 256 + ooff + n], x)


def test_stream_pieces_take_fast_kernel(b64):
    """A streaming decode in large odd-sized pieces (every piece's quads misaligned): the result
    equals the oracle's one-shot decode, and the pieces' bulk runs through dec_fastu_kernel (one
    launch per piece: the join rides along)."""
    x = synth.data(3_000_001, seed=4)
    ref = oracle.encode(x)
    td = torch.from_numpy(ref).to(DEV)
    for piece in (100_003, 300_001):  # (pieces' bulk >= 64 Ki chars: the unaligned fast kernel)
        ds = b64.DecodeStream()
        before = b64.launch_count()
        parts, p = [], 0
        while p < ref.size:
            k = min(piece, ref.size - p)
            parts.append(ds.update(td[p: p + k]))
            p += k
        npieces = len(parts)
        tail, info = ds.end()
        torch.cuda.synchronize()
        launches = b64.launch_count() - before
        err, st, olen = info.tolist()
        got = torch.cat(parts + [tail]).cpu().numpy()
        assert err == -1 and olen == x.size and np.array_equal(got[: x.size], x)
        assert launches <= npieces + 1, (launches, npieces)


def test_decode_misaligned_every_phase(b64):
    """Every input offset mod 32 x every output offset mod 8 (all 8 word shifts x 4 byte shifts
    of dec_fastu_kernel, and every head-quad count) at one size, against the oracle."""
    n = 150_001
    x = synth.data(n, seed=11)
    ref = oracle.encode(x)
    m = ref.size
    src = torch.from_numpy(ref).to(DEV)
    tb = torch.empty(m + 64, dtype=torch.uint8, device=DEV)
    ob = torch.empty(3 * (m // 4) + 64, dtype=torch.uint8, device=DEV)
    xd = torch.from_numpy(x).to(DEV)
    for ioff in range(32):
        tin = tb[ioff: ioff + m]
        tin.copy_(src)
        for ooff in range(8):
            out = ob[ooff: ooff + 3 * (m // 4)]
            y, info = b64.decode_async(tin, out=out)
            err, st, olen = info.tolist()
            assert err == -1 and olen == n, (ioff, ooff)
            assert torch.equal(y[:n], xd), (ioff, ooff)


# ------------------------------------------------------------------ whitespace decode, general path (large)

def _wrap(text, every, seed, extra_ws=b"\r\n"):
    rng = np.random.default_rng(seed)
    parts, i = [], 0
    while i < text.size:
        k = int(rng.integers(1, 2 * every))
        parts.append(text[i: i + k])
        parts.append(np.frombuffer(extra_ws[: int(rng.integers(1, len(extra_ws) + 1))], np.uint8))
        i += k
    return np.concatenate(parts)


@pytest.mark.parametrize("alpha_kind", ["std", "ws_data"])
def test_decode_ws_general_path_large(b64, alpha_kind):
    """Texts above the single-launch size with irregular whitespace runs: the general path
    (count / scan / compaction / decode / finalize), with the arithmetic whitespace test (std)
    and with the table test (an alphabet in which ' ' and TAB are data chars); valid, with an
    error, and with a compacted length that is not a multiple of 4."""
    if alpha_kind == "std":
        chars, alpha, ws = oracle.STANDARD, b64.standard(), b"\r\n\t \x0b\x0c"
    else:
        chars = oracle.STANDARD[:62] + b" \t"
        alpha, ws = b64.alphabet(chars), b"\r\n\x0b\x0c"
    for n in (700_001, 3_000_000):
        x = synth.data(n, seed=n)
        text = oracle.encode(x, chars)
        # (the 4th layout: whitespace runs of up to 200 bytes -- words, lanes and whole 128-byte
        # rows with nothing kept, which the compaction's branch-free stores send to a scratch word)
        long_ws = ws[:2] * 100
        for v, t in enumerate((_wrap(text, 60, n, ws), _wrap(text, 7, n + 1, ws), _wrap(text[:-1], 30, n + 2, ws),
                               _wrap(text, 40, n + 3, long_ws))):
            if v == 0:
                t = t.copy()
                t[t.size // 3] = ord("*")
            ref, rerr, rst = oracle.decode_ws(t, chars)
            out, err = b64.decode_ws(torch.from_numpy(t).to(DEV), alpha)
            assert err == rerr, (n, v, err, rerr)
            assert np.array_equal(out.cpu().numpy(), ref), (n, v)


# ------------------------------------------------------------------ whitespace decode: line segments

def _mime_lines(text, L, sep=b"\r\n"):
    lines = [text[i: i + L] for i in range(0, text.size, L)]
    out = []
    for ln in lines:
        out.append(ln)
        out.append(np.frombuffer(sep, np.uint8))
    return np.concatenate(out)


def _insert(t, pos, b):
    return np.concatenate([t[:pos], np.frombuffer(b, np.uint8), t[pos:]])


def _varying(m, lens=(60, 72, 84, 76)):
    i, k = 0, 0
    while i < m:
        yield i, lens[k % len(lens)]
        i += lens[k % len(lens)]
        k += 1


def test_decode_ws_line_segments(b64):
    """Line-structured text whose layout breaks (a stray blank, a missing or doubled line break,
    a change of line length): the line pass keeps the verified blocks, probes the rest again
    (up to 3 segments) and hands what is left to the general path -- every variant against
    the oracle (error offset in the ORIGINAL text, status, exact bytes), with errors before,
    inside and after the break and LENGTH texts."""
    n = 2_000_000
    x = synth.data(n, seed=33)
    t = oracle.encode(x)
    mime = _mime_lines(t, 76)
    M = mime.size
    cases = {
        "blank_middle": _insert(mime, M // 2, b" "),
        "blank_start": _insert(mime, 200, b" "),
        "blank_end": _insert(mime, M - 5000, b" "),
        "two_blanks": _insert(_insert(mime, M // 3, b" "), 2 * M // 3, b"\t"),
        "four_blanks": _insert(_insert(_insert(_insert(mime, M // 5, b" "), 2 * M // 5, b" "), 3 * M // 5, b" "),
                               4 * M // 5, b" "),
        "missing_crlf": np.concatenate([mime[: 78 * 9000 + 76], mime[78 * 9000 + 78:]]),
        "double_crlf": _insert(mime, 78 * 12000, b"\r\n"),
        "relayout": np.concatenate([_mime_lines(t[: 76 * 10000], 76), _mime_lines(t[76 * 10000:], 64, b"\n")]),
        "block_boundary": _insert(mime, (4096 // 76) * 78 * 3, b" "),
        # no uniform layout (lines of 60 / 72 / 84 / 76 chars in turn): the first segment and
        # the reprobed one break in their first block, and the general path takes the rest
        "varying_lines": np.concatenate([np.concatenate([t[i: i + L], np.frombuffer(b"\n", np.uint8)])
                                         for i, L in _varying(t.size)]),
    }
    for name, tv in list(cases.items()):
        cases[name + "+err_before"] = tv.copy()
        cases[name + "+err_before"][1000] = ord("*")
        c2 = tv.copy()
        c2[tv.size - 3000] = ord("#")
        cases[name + "+err_after"] = c2
    cases["blank_middle+length"] = _insert(_mime_lines(t[:-1], 76), M // 2, b" ")
    cases["blank_middle+err_at_blank"] = _insert(mime, M // 2, b"*")
    for name, tv in cases.items():
        ref, rerr, rst = oracle.decode_ws(tv)
        out, info = None, None
        o, err = b64.decode_ws(torch.from_numpy(tv).to(DEV))
        assert err == rerr, (name, err, rerr)
        assert np.array_equal(o.cpu().numpy(), ref), name


def test_decode_ws_line_path_ragged_end(b64):
    """The line kernel's last step: its kept chars end anywhere in a 32-char unit (the unit
    loads past them read filler, not stale chars), with an incomplete final group (LENGTH),
    an invalid char or a pad in it, an error in the last full quad, and a final line of every
    length mod 4 -- against the oracle (error offset in the original text, exact bytes)."""
    x = synth.data(600_000, seed=71)
    t = oracle.encode(x)
    tails = {"len0": b"", "AB": b"AB", "ABC": b"ABC", "A": b"A", "A*": b"A*", "*B": b"*B", "A=": b"A=",
             "AB=": b"AB=", "AB C": b"AB C", "ABCD": b"ABCD", "AB*D": b"AB*D"}
    for cut in (0, 4, 36, 72, 1000):
        body = t[: t.size - cut]
        for name, tail in tails.items():
            tv = np.concatenate([body, np.frombuffer(tail, np.uint8)])
            mime = _mime_lines(tv, 76)
            ref, rerr, rst = oracle.decode_ws(mime)
            o, err = b64.decode_ws(torch.from_numpy(mime).to(DEV))
            assert err == rerr, (cut, name, err, rerr)
            assert np.array_equal(o.cpu().numpy(), ref), (cut, name)


# ------------------------------------------------------------------ decode -> consumer (f3)

def test_decode_consume_vs_oracle(b64):
    """b64_decode_consume: chunks decoded into a small ring and handed to a consumer that copies
    them out -- the reassembled output, err_off and out_len equal the oracle's (valid text with
    every pad count, an error in the middle chunk, a text shorter than one chunk)."""
    for n, bad_at in ((3_000_001, None), (3_000_002, 1_500_003), (1_234, None), (3_000_000, None)):
        x = synth.data(n, seed=n)
        t = oracle.encode(x)
        if bad_at is not None:
            t = t.copy()
            t[bad_at] = ord("!")
        ref, rerr, _ = oracle.decode(t)
        full = torch.zeros(b64.decoded_len_max(t.size), dtype=torch.uint8, device=DEV)
        seen = []

        def consumer(chunk, off):
            full[off: off + chunk.numel()].copy_(chunk)
            seen.append((off, chunk.numel()))

        err, olen = b64.decode_consume(torch.from_numpy(t).to(DEV), consumer, ring_bytes=1 << 20)
        assert err == rerr and olen == ref.size, (n, err, rerr, olen)
        assert np.array_equal(full[:olen].cpu().numpy(), ref), n
        assert sum(k for _, k in seen) == full.numel() and [o for o, _ in seen] == sorted(o for o, _ in seen)


def test_decode_consume_sum(b64):
    """A reducing consumer (the decoded bytes never leave L2): the per-chunk sums add up to the
    sum of the oracle's decode."""
    x = synth.data(20_000_004, seed=9)  # n % 3 == 0: no padding, every decoded byte is data
    x = x[:20_000_004 - 20_000_004 % 3]
    t = torch.from_numpy(oracle.encode(x)).to(DEV)
    acc = torch.zeros(1, dtype=torch.int64, device=DEV)
    err, olen = b64.decode_consume(t, lambda c, off: acc.add_(c.sum(dtype=torch.int64)), ring_bytes=8 << 20)
    assert err == -1 and olen == x.size
    assert int(acc.item()) == int(x.sum(dtype=np.int64))


def test_batch_fast_path_many_errors(b64):
    """So many corrupted windows that a warp's note list of the bulk pass overflows (the per-string
    fallback then redoes the batch): results still equal the oracle's; and a moderately corrupted
    batch (reported from the notes) too."""
    text, toff = _batch_case(20000, seed=23, hi=600)
    count = toff.size - 1
    rng = np.random.default_rng(23)
    for frac in (0.02, 0.6):
        t = text.copy()
        for s in rng.choice(count, int(frac * count), replace=False):
            L = toff[s + 1] - toff[s]
            for _ in range(3):
                t[toff[s] + rng.integers(0, L)] = ord("!")
        rout, roff, rst, rerr, rlen = oracle.decode_batch(t, toff)
        out, oo, st, err, olen = b64.decode_batch(torch.from_numpy(t).to(DEV), torch.from_numpy(toff).to(DEV))
        assert np.array_equal(st.cpu().numpy(), rst), frac
        assert np.array_equal(err.cpu().numpy(), rerr), frac
        assert np.array_equal(olen.cpu().numpy(), rlen), frac


def _stream_into(b64, dt, alpha, pieces, overlap):
    """Decode dt in the given pieces into ONE preallocated buffer (no host sync and no other
    launch between the updates, so the overlap mode really overlaps)."""
    ds = b64.DecodeStream(alpha, overlap=overlap)
    buf = torch.full((3 * (dt.numel() // 4) + 16,), 0xA5, dtype=torch.uint8, device=DEV)
    o = p = 0
    for k in pieces:
        n = ds.out_len(k)
        got = ds.update(dt[p: p + k], out=buf[o: o + max(n, 1)])
        assert got.numel() == n
        o += n
        p += k
    tail, info = ds.end(out=buf[o: o + max(ds.end_len(), 1)])
    return buf, info.tolist()


@pytest.mark.parametrize("ai", [0, 1, 3, 4])
def test_stream_overlap_vs_oracle(b64, ai):
    """B64_STREAM_OVERLAP (each piece's bulk runs while the previous piece drains): for large
    pieces of odd and aligned sizes, texts with bad chars in several pieces (the first one is the
    error), a bad final quad and a LENGTH tail, the result equals the oracle's one-shot decode and
    the default mode's, bit for bit; repeated to give a race a chance."""
    perm = np.random.default_rng(7).permutation(127)[:65]
    al = [(oracle.STANDARD, oracle.PAD, b64.standard()), (oracle.URL, oracle.PAD, b64.url()), None,
          (bytes(perm[:64].tolist()), int(perm[64]), b64.alphabet(bytes(perm[:64].tolist()), bytes([int(perm[64])]))),
          (oracle.STANDARD, oracle.PAD, b64.lenient_of(b64.standard()))]
    chars, pad, alpha = al[ai]
    rng = np.random.default_rng(70 + ai)
    x = synth.data(6_000_001 + ai, seed=70 + ai)
    text = oracle.encode(x, chars, pad)
    variants = [text]
    t2 = text.copy()
    for p_ in sorted(rng.choice(text.size - 8, 3, replace=False))[::-1]:  # bad chars in 3 places
        t2[p_] = ord("*")
    variants.append(t2)
    t3 = text.copy()
    t3[-1] = ord("!")
    variants.append(t3)
    variants.append(text[:-2])  # LENGTH
    for v in variants:
        ref, rerr, rst = oracle.decode(v, chars, pad, lenient=(ai == 4))
        dt = torch.from_numpy(v).to(DEV)
        for pieces in ([(1 << 20) + 3] * (v.size // ((1 << 20) + 3)) + [v.size % ((1 << 20) + 3)],
                       [1 << 20] * (v.size // (1 << 20)) + [v.size % (1 << 20)],
                       None):
            if pieces is None:
                cuts = np.sort(rng.choice(np.arange(70_000, v.size - 70_000), 5, replace=False))
                pieces = np.diff(np.concatenate([[0], cuts, [v.size]])).tolist()
            base, binfo = _stream_into(b64, dt, alpha, pieces, overlap=False)
            for rep in range(3):
                got, info = _stream_into(b64, dt, alpha, pieces, overlap=True)
                err, st, olen = info
                assert (err, st) == (rerr, rst) and info == binfo, (ai, rep, info, binfo, rerr, rst)
                assert torch.equal(got, base)
                if err < 0:
                    assert olen == ref.size and np.array_equal(got[:olen].cpu().numpy(), ref)


@pytest.mark.parametrize("n", [150_000, 150_001, 150_002, 1_000_003])
def test_encode_misaligned_every_phase(b64, n):
    """Every input offset mod 8 x every 4-byte-aligned output offset mod 32 (all shifts of
    enc_fastu_kernel and every head-triple count q0 = 0..7), plus an output that is not 4-byte
    aligned (the byte-store generic path), against the oracle; the bytes around the output
    are untouched."""
    x = synth.data(n, seed=n)
    ref = oracle.encode(x)
    m = ref.size
    xb = torch.empty(n + 64, dtype=torch.uint8, device=DEV)
    ob = torch.empty(m + 128, dtype=torch.uint8, device=DEV)
    xd = torch.from_numpy(x).to(DEV)
    for ioff in range(8):
        xin = xb[ioff: ioff + n]
        xin.copy_(xd)
        for ooff in list(range(0, 32, 4)) + [3]:
            ob.fill_(0xA5)
            out = b64.encode(xin, out=ob[32 + ooff: 32 + ooff + m])
            assert out.numel() == m
            h = ob.cpu().numpy()
            assert (h[: 32 + ooff] == 0xA5).all() and (h[32 + ooff + m:] == 0xA5).all(), (ioff, ooff)
            assert np.array_equal(h[32 + ooff: 32 + ooff + m], ref), (n, ioff, ooff)


def test_encode_stream_large_pieces(b64):
    """A streaming encode in large pieces of odd and aligned sizes (the pieces' bulk through
    enc_fastu_kernel when misaligned, enc_fast_kernel when aligned, with 0-2 held bytes at the
    boundaries): the concatenation equals the oracle's one-shot encode."""
    x = synth.data(3_000_001, seed=5)
    ref = oracle.encode(x)
    xd = torch.from_numpy(x).to(DEV)
    for piece in (100_001, 300_002, 262_144, 65_536 * 3):
        es = b64.EncodeStream()
        parts, p = [], 0
        while p < x.size:
            k = min(piece, x.size - p)
            parts.append(es.update(xd[p: p + k]))
            p += k
        parts.append(es.end())
        got = torch.cat(parts).cpu().numpy()
        assert np.array_equal(got, ref), piece


@pytest.mark.parametrize("ai", [0, 1, 3])
def test_encode_stream_overlap_vs_oracle(b64, ai):
    """B64_STREAM_OVERLAP for the streaming encode (each piece's bulk runs while the previous
    piece drains; the join with the held bytes at the kernel's end): pieces of odd, aligned and
    random sizes, written into ONE buffer with no launch in between, equal the oracle's one-shot
    encode and the default mode's output, repeated to give a race a chance."""
    perm = np.random.default_rng(7).permutation(127)[:65]
    al = [(oracle.STANDARD, oracle.PAD, b64.standard()), (oracle.URL, oracle.PAD, b64.url()), None,
          (bytes(perm[:64].tolist()), int(perm[64]), b64.alphabet(bytes(perm[:64].tolist()), bytes([int(perm[64])])))]
    chars, pad, alpha = al[ai]
    rng = np.random.default_rng(90 + ai)
    x = synth.data(5_000_002 + ai, seed=90 + ai)
    ref = oracle.encode(x, chars, pad)
    xd = torch.from_numpy(x).to(DEV)
    cuts = np.sort(rng.choice(np.arange(70_000, x.size - 70_000), 5, replace=False))
    for pieces in ([(1 << 20) + 1] * (x.size // ((1 << 20) + 1)) + [x.size % ((1 << 20) + 1)],
                   [3 << 18] * (x.size // (3 << 18)) + [x.size % (3 << 18)],
                   np.diff(np.concatenate([[0], cuts, [x.size]])).tolist()):
        outs = []
        for overlap in (False, True, True, True):
            es = b64.EncodeStream(alpha, overlap=overlap)
            buf = torch.full((ref.size + 16,), 0xA5, dtype=torch.uint8, device=DEV)
            o = p = 0
            for k in pieces:
                c = es.out_len(k)
                got = es.update(xd[p: p + k], out=buf[o: o + max(c, 1)])
                assert got.numel() == c
                o += c
                p += k
            es.end(out=buf[o: o + max(es.end_len(), 1)])
            outs.append(buf)
        for b in outs:
            assert torch.equal(b, outs[0])
        h = outs[0].cpu().numpy()
        assert np.array_equal(h[: ref.size], ref) and (h[ref.size:] == 0xA5).all(), (ai, pieces[:2])


def test_decode_ws_general_path_errors_across_tiles(b64):
    """The general path (count / scan / compaction over 4 KiB chunks grouped per CTA) and its
    error mapping: one bad char at a time in the first chunk, at 32 KiB, deep in the middle and
    in the last chunks of a 2.5 MB irregular text; a whitespace-only tail of several chunks; the
    same texts decoded twice in a row."""
    x = synth.data(1_900_003, seed=61)
    text = oracle.encode(x)
    t = _wrap(text, 45, 61, b"\r\n \t")
    tile = 8 * 4096
    keep = np.nonzero(~np.isin(t, np.frombuffer(b"\r\n \t", np.uint8)))[0]
    for target in (5, tile - 1, tile, 3 * tile + 17, t.size // 2, t.size - 40):
        p = int(keep[np.searchsorted(keep, target)])
        t2 = t.copy()
        t2[p] = ord("%")
        ref, rerr, rst = oracle.decode_ws(t2)
        for _ in range(2):
            out, err = b64.decode_ws(torch.from_numpy(t2).to(DEV))
            assert err == rerr == p, (target, err, rerr)
            assert np.array_equal(out.cpu().numpy(), ref)
    t3 = np.concatenate([t, np.frombuffer(b" \r\n\t" * 5000, np.uint8)])  # 20 KB of trailing whitespace
    ref, rerr, _ = oracle.decode_ws(t3)
    out, err = b64.decode_ws(torch.from_numpy(t3).to(DEV))
    assert err == rerr == -1 and np.array_equal(out.cpu().numpy(), ref)


def test_stream_overlap_errors_at_piece_boundaries(b64):
    """Overlap mode: a bad char at a piece's first char (the join quad, decoded after the wait
    by the EARLY kernel's last thread), at its last char (held back for the next piece) or in
    the middle of a later piece (the bulk's error path, which waits before its atomicMin): the
    reported first error is the oracle's every time, in both modes."""
    x = synth.data(4_500_000, seed=91)
    text = oracle.encode(x)
    piece = (1 << 20) + 1
    cuts = list(range(0, text.size, piece))
    for where in ("first", "last", "mid"):
        for k in (1, 3):
            t = text.copy()
            if where == "first":
                p = cuts[k]
            elif where == "last":
                p = cuts[k + 1] - 1
            else:
                p = cuts[k] + piece // 2
            t[p] = ord("?")
            dt = torch.from_numpy(t).to(DEV)
            pieces = [min(piece, t.size - c) for c in cuts]
            ref, rerr, rst = oracle.decode(t)
            assert rerr == p
            for overlap in (False, True):
                _, info = _stream_into(b64, dt, b64.standard(), pieces, overlap=overlap)
                assert info[:2] == [rerr, rst], (where, k, overlap, info, rerr)
