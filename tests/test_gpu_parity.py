"""GPU parity: the CUDA path (through the C ABI) vs the oracle, bit-exact.

Every comparison is element by element on the same seeded inputs (synth/):
encoded chars, decoded bytes (the exact prefix on error), err_off, status and
out_len.  Sizes span several warp-chunks (768 B / 1024 chars) with ragged
tails, misaligned pointers (the generic kernels), every byte value at every
position of small texts, and BASELINE.json's configs at full size (sampled
windows where the oracle would need more host memory than is sensible).
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


def _alphabets(b64):
    rng = np.random.default_rng(7)
    out = [(oracle.STANDARD, oracle.PAD, b64.standard()), (oracle.URL, oracle.PAD, b64.url())]
    while len(out) < 7:
        perm = rng.permutation(127)[:65]
        chars, pad = bytes(perm[:64].tolist()), int(perm[64])
        out.append((chars, pad, b64.alphabet(chars, bytes([pad]))))
    return out


def to_dev(x: np.ndarray, offset: int = 0) -> torch.Tensor:
    """Copy to the device at a chosen byte misalignment (offset) inside a fresh buffer."""
    buf = torch.empty(x.size + offset + 64, dtype=torch.uint8, device=DEV)
    t = buf[offset: offset + x.size]
    if x.size:
        t.copy_(torch.from_numpy(x))
    return t


def dec_check(b64, text: np.ndarray, chars, pad, alpha, off_in=0, off_out=0):
    t = to_dev(text, off_in)
    cap = 3 * (text.size // 4)
    obuf = torch.empty(cap + off_out + 64, dtype=torch.uint8, device=DEV)
    out, info = b64.decode_async(t, alpha, out=obuf[off_out: off_out + max(cap, 1)])
    err, st, olen = info.tolist()
    ref, rerr, rst = oracle.decode(text, chars, pad)
    assert (err, st) == (rerr, rst), (err, st, rerr, rst)
    assert olen == ref.size
    assert np.array_equal(out[:olen].cpu().numpy(), ref)
    return err


# ------------------------------------------------------------------ generator twin

def test_synth_device_matches_host(b64):
    for n, off in ((0, 0), (1, 0), (7, 3), (4096, 0), (100003, 5), (1 << 20, 13), (3000, 1 << 33)):
        d = torch.empty(n + 16, dtype=torch.uint8, device=DEV)
        for shift in (0, 3):
            t = d[shift: shift + n]
            synth.device_fill(t, seed=0, offset=off)
            assert np.array_equal(t.cpu().numpy(), synth.data(n, 0, off)), (n, off, shift)


# ------------------------------------------------------------------ encode

def test_encode_fuzz_lengths(b64):
    al = _alphabets(b64)
    for n in range(0, 4097):
        chars, pad, alpha = al[n % len(al)]
        x = synth.data(n, seed=n)
        t = b64.encode(to_dev(x), alpha)
        assert np.array_equal(t.cpu().numpy(), oracle.encode(x, chars, pad)), n


def test_encode_chunk_boundaries(b64):
    for k in (1, 2, 3, 37, 148 * 8, 148 * 8 * 2 + 5):
        for r in range(0, 24):
            n = 768 * k + r
            x = synth.data(n, seed=k * 100 + r)
            t = b64.encode(to_dev(x))
            assert np.array_equal(t.cpu().numpy(), oracle.encode(x)), n


def test_encode_misaligned_generic(b64):
    al = _alphabets(b64)
    for i, n in enumerate((1, 2, 11, 12, 13, 100, 767, 768, 769, 5000, 100003)):
        for oi in (0, 1, 2, 3, 5):
            for oo in (0, 1, 2, 4, 16):
                if oi == 0 and oo == 0:
                    continue
                chars, pad, alpha = al[(i + oi + oo) % len(al)]
                x = synth.data(n, seed=n + oi)
                obuf = torch.empty(b64.encoded_len(n) + oo + 64, dtype=torch.uint8, device=DEV)
                t = b64.encode(to_dev(x, oi), alpha, out=obuf[oo:])
                assert np.array_equal(t.cpu().numpy(), oracle.encode(x, chars, pad)), (n, oi, oo)


# ------------------------------------------------------------------ decode

def test_decode_fuzz_valid_and_corrupted(b64):
    al = _alphabets(b64)
    for n in range(0, 3100, 7):
        chars, pad, alpha = al[n % len(al)]
        x = synth.data(n, seed=n)
        text = oracle.encode(x, chars, pad)
        assert dec_check(b64, text, chars, pad, alpha) == -1
        if text.size:
            k = 1 + n % 3
            pos, bad = synth.corruption(min(k, text.size), text.size, chars, seed=n, pad=pad)
            t2 = text.copy()
            t2[pos] = bad
            assert dec_check(b64, t2, chars, pad, alpha) == int(pos.min())
            # non-ASCII bytes and a misplaced pad are invalid too
            t3 = text.copy()
            p = int(pos[0])
            t3[p] = 0x80 | (n & 0x7F)
            dec_check(b64, t3, chars, pad, alpha)
            if p < text.size - 4:
                t3[p] = pad
                assert dec_check(b64, t3, chars, pad, alpha) == p


def test_decode_every_byte_every_position(b64):
    """Exhaustive substitution on small texts (interior + all final-quad forms)."""
    std = b64.standard()
    for raw_len in (30, 31, 32):  # final quad 'xxxx', 'xx==', 'xxx='
        text = oracle.encode(synth.data(raw_len, seed=raw_len))
        for p in range(text.size):
            for v in range(256):
                t = text.copy()
                t[p] = v
                dec_check(b64, t, oracle.STANDARD, oracle.PAD, std)


def test_decode_chunk_boundaries_and_errors(b64):
    std = b64.standard()
    for k in (1, 2, 5, 148 * 8 + 3):
        for r in (0, 4, 8, 1020):
            m_raw = (1024 * k + r) // 4 * 3 - (k % 3)
            x = synth.data(m_raw, seed=k + r)
            text = oracle.encode(x)
            dec_check(b64, text, oracle.STANDARD, oracle.PAD, std)
            for j in range(4):
                pos, bad = synth.corruption(1 + j, text.size, oracle.STANDARD, seed=100 * k + r + j)
                t2 = text.copy()
                t2[pos] = bad
                dec_check(b64, t2, oracle.STANDARD, oracle.PAD, std)
            # error in the last char of a warp-chunk / the very last char
            for p in {1023, min(text.size - 1, 2047), text.size - 5, text.size - 1}:
                if 0 <= p < text.size:
                    t2 = text.copy()
                    t2[p] = ord("*")
                    dec_check(b64, t2, oracle.STANDARD, oracle.PAD, std)


def test_decode_misaligned_generic(b64):
    al = _alphabets(b64)
    for i, n in enumerate((0, 1, 2, 3, 4, 12, 13, 47, 48, 49, 767, 768, 4000, 100001)):
        chars, pad, alpha = al[i % len(al)]
        text = oracle.encode(synth.data(n, seed=n), chars, pad)
        for oi in (0, 1, 3, 4, 16):
            for oo in (0, 1, 2, 3, 8):
                if oi == 0 and oo == 0:
                    continue
                dec_check(b64, text, chars, pad, alpha, oi, oo)
                if text.size > 8:
                    pos, bad = synth.corruption(2, text.size, chars, seed=n + oi + oo, pad=pad)
                    t2 = text.copy()
                    t2[pos] = bad
                    dec_check(b64, t2, chars, pad, alpha, oi, oo)


def test_decode_length_error_sync(b64):
    with pytest.raises(b64.B64Error, match="ELENGTH"):
        b64.decode(torch.zeros(5, dtype=torch.uint8, device=DEV))
    out, err = b64.decode(torch.zeros(0, dtype=torch.uint8, device=DEV))
    assert err == -1 and out.numel() == 0


def test_decode_chunk_api_shards(b64):
    """b64_decode_chunk over shards at arbitrary 4-char boundaries + device MIN == oracle."""
    std = b64.standard()
    x = synth.data(300_001, seed=5)
    text = oracle.encode(x)
    m = text.size
    for trial in range(6):
        t2 = text.copy()
        if trial:
            pos, bad = synth.corruption(trial, m, oracle.STANDARD, seed=trial)
            t2[pos] = bad
        ref, rerr, rst = oracle.decode(t2)
        Q = m // 4
        cuts = sorted({0, Q} | {int(q) for q in synth.words(9, 9, trial * 8, 5) % Q})
        dt = to_dev(t2)
        out = torch.empty(3 * Q, dtype=torch.uint8, device=DEV)
        cells = torch.full((len(cuts) - 1,), b64.ERR_NONE, dtype=torch.int64, device=DEV)
        for i in range(len(cuts) - 1):
            a, b = 4 * cuts[i], 4 * cuts[i + 1]
            b64.decode_chunk(dt[a:b], a, b == m, cells[i: i + 1], std, out=out[3 * cuts[i]: 3 * cuts[i + 1]])
        cell = cells.min().reshape(1)
        eo = torch.empty(1, dtype=torch.int64, device=DEV)
        st = torch.zeros(1, dtype=torch.int32, device=DEV)
        b64.decode_finalize(cell, eo, st)
        assert (int(eo.item()), int(st.item())) == (rerr, rst)
        assert np.array_equal(out[: ref.size].cpu().numpy(), ref)


# ------------------------------------------------------------------ batched

def _batch_case(count, hi, seed, corrupt_frac=0.01):
    L = synth.loguniform_lengths(count, hi=hi, seed=seed)
    off = synth.offsets(L)
    x = synth.data(int(off[-1]), seed=seed)
    return L, off, x


def test_batch_encode_decode_vs_oracle(b64):
    for count, hi, seed in ((1, 10, 1), (7, 100, 2), (5000, 65536, 3), (20000, 4096, 4)):
        L, off, x = _batch_case(count, hi, seed)
        doff = torch.from_numpy(off).to(DEV)
        enc, eoff = b64.encode_batch(to_dev(x), doff)
        renc, reoff = oracle.encode_batch(x, off)
        assert np.array_equal(eoff.cpu().numpy(), reoff)
        assert np.array_equal(enc[: reoff[-1]].cpu().numpy(), renc)
        # corrupt ~1% of strings (seeded), plus a few length errors
        text = renc.copy()
        tl = np.diff(reoff)
        picks = synth.pick(count, 0.01, seed=seed)
        for i in picks:
            if tl[i]:
                pos, bad = synth.corruption(1, int(tl[i]), oracle.STANDARD, seed=int(i))
                text[reoff[i] + pos] = bad
        din = reoff.copy()
        if count > 3:  # make string 1 end mid-quad: shift the boundary by 1
            din[2] -= 1 if tl[1] > 0 else 0
        out, ooff, st, err, olen = b64.decode_batch(to_dev(text), torch.from_numpy(din).to(DEV))
        rout, rooff, rst, rerr, rolen = oracle.decode_batch(text, din)
        assert np.array_equal(ooff.cpu().numpy(), rooff)
        assert np.array_equal(st.cpu().numpy(), rst)
        assert np.array_equal(err.cpu().numpy(), rerr)
        assert np.array_equal(olen.cpu().numpy(), rolen)
        o = out.cpu().numpy()
        for i in range(count):
            assert np.array_equal(o[rooff[i]: rooff[i] + rolen[i]], rout[rooff[i]: rooff[i] + rolen[i]]), i


def test_batch_sharded_single_gpu(b64):
    """configs[3]'s multi-GPU form on one GPU: the batch cut into W shards by cumulative bytes
    (dist.batch_shard), each decoded through b64_decode_batch_ex with offsets that are a SLICE of
    the whole batch's (first offset > 0, same buffer) and its global first string index; the
    shards' first-failing words MIN-combined equal the whole batch's first failing string, and
    every per-string result equals the oracle's."""
    from paper_1910_05109_b200 import dist as b64dist

    count = 30_000
    L, off, x = _batch_case(count, 65536, 11)
    renc, reoff = oracle.encode_batch(x, off)
    text = renc.copy()
    tl = np.diff(reoff)
    picks = synth.pick(count, 0.01, seed=12)
    for i in picks:
        if tl[i]:
            pos, bad = synth.corruption(1, int(tl[i]), oracle.STANDARD, seed=int(i))
            text[reoff[i] + pos] = bad
    rout, rooff, rst, rerr, rolen = oracle.decode_batch(text, reoff)
    want_first = int(np.flatnonzero(rst)[0]) if np.any(rst) else -1
    dt, dx = to_dev(text), to_dev(x)
    doff_t, doff_x = torch.from_numpy(reoff).to(DEV), torch.from_numpy(off).to(DEV)
    for W in (1, 2, 3, 8):
        cells = torch.full((W,), b64.ERR_NONE, dtype=torch.int64, device=DEV)
        for r in range(W):
            es = b64dist.batch_shard(off, W, r)
            eo, eoo = b64.encode_batch(dx, doff_x[es.start: es.stop + 1])
            assert np.array_equal(eo[: int(eoo[-1])].cpu().numpy(), renc[reoff[es.start]: reoff[es.stop]]), (W, r)
            ds = b64dist.batch_shard(reoff, W, r)
            out, ooff, st, err, olen = b64.decode_batch(dt, doff_t[ds.start: ds.stop + 1], index_base=ds.start,
                                                        first_bad=cells[r:r + 1])
            assert np.array_equal(st.cpu().numpy(), rst[ds.start: ds.stop]), (W, r)
            assert np.array_equal(err.cpu().numpy(), rerr[ds.start: ds.stop]), (W, r)
            assert np.array_equal(olen.cpu().numpy(), rolen[ds.start: ds.stop]), (W, r)
            o, oo = out.cpu().numpy(), ooff.cpu().numpy()
            for j in range(0, ds.stop - ds.start, 97):
                i = ds.start + j
                assert np.array_equal(o[oo[j]: oo[j] + rolen[i]], rout[rooff[i]: rooff[i] + rolen[i]]), (W, i)
        v = int(cells.min().item())
        assert (v if v < b64.ERR_NONE else -1) == want_first, W
    # no failing string: the word stays untouched
    clean = torch.full((1,), b64.ERR_NONE, dtype=torch.int64, device=DEV)
    b64.decode_batch(to_dev(renc), torch.from_numpy(reoff).to(DEV), index_base=5, first_bad=clean)
    assert int(clean.item()) == b64.ERR_NONE


def test_batch_many_short_strings(b64):
    """200k strings of 0..140 bytes (the lane-per-string path and its hand-over to the warp path
    at the thresholds, strings straddling warp ranges), ~5 % corrupted anywhere (interior and
    final-quad chars, '=' misplaced), a few LENGTH errors; strict and lenient alphabets."""
    count = 200_000
    L = (synth.words(77, 3, 0, count) % np.uint64(141)).astype(np.int64)
    off = synth.offsets(L)
    x = synth.data(int(off[-1]), seed=77)
    doff = torch.from_numpy(off).to(DEV)
    enc, eoff = b64.encode_batch(to_dev(x, 1), doff)  # misaligned input base too
    renc, reoff = oracle.encode_batch(x, off)
    assert np.array_equal(eoff.cpu().numpy(), reoff)
    assert np.array_equal(enc[: reoff[-1]].cpu().numpy(), renc)
    text = renc.copy()
    tl = np.diff(reoff)
    picks = synth.pick(count, 0.05, seed=78)
    w = synth.words(79, 3, 0, len(picks))
    for k, i in enumerate(picks):
        if tl[i]:
            p = int(w[k] % np.uint64(tl[i]))
            text[reoff[i] + p] = (ord("="), ord("*"), 0xC3)[k % 3]
    din = reoff.copy()
    for i in range(5, count, 997):  # shift some boundaries: LENGTH errors on both sides
        if din[i] + 1 <= din[i + 1]:  # offsets stay non-decreasing (the API's precondition)
            din[i] += 1
    for alpha, lenient in ((b64.standard(), False), (b64.lenient_of(b64.standard()), True)):
        out, ooff, st, err, olen = b64.decode_batch(to_dev(text, 3), torch.from_numpy(din).to(DEV), alpha)
        rout, rooff, rst, rerr, rolen = oracle.decode_batch(text, din, lenient=lenient)
        assert np.array_equal(st.cpu().numpy(), rst)
        assert np.array_equal(err.cpu().numpy(), rerr)
        assert np.array_equal(olen.cpu().numpy(), rolen)
        o = out.cpu().numpy()
        for i in np.flatnonzero(rolen):
            assert np.array_equal(o[rooff[i]: rooff[i] + rolen[i]], rout[rooff[i]: rooff[i] + rolen[i]]), i


def test_batch_misaligned_offsets(b64):
    """String starts at every alignment: input offsets shifted by a 1..3 byte prefix gap."""
    for gap in (1, 2, 3):
        L = np.array([0, 1, 2, 3, 4, 5, 47, 48, 49, 100, 0, 767, 1024, 3000, 1], dtype=np.int64)
        Lg = L + gap
        off = synth.offsets(Lg)
        x = synth.data(int(off[-1]), seed=gap)
        in_off = off.copy()
        in_off[:-1] += gap  # each string starts gap bytes into its slot
        starts, ends = in_off[:-1], off[1:]
        # encode: strings [starts[i], ends[i])
        # (offsets must be non-decreasing: represent as pairs via interleaved empty strings)
        pairs = np.empty(2 * len(L) + 1, dtype=np.int64)
        pairs[0] = 0
        pairs[1::2] = starts
        pairs[2::2] = ends
        enc, eoff = b64.encode_batch(to_dev(x), torch.from_numpy(pairs).to(DEV))
        renc, reoff = oracle.encode_batch(x, pairs)
        assert np.array_equal(enc[: reoff[-1]].cpu().numpy(), renc)
        # decode the encoded strings placed back at odd offsets
        tl = np.diff(reoff)
        text = np.concatenate([np.concatenate([np.full(gap, ord("A"), np.uint8), renc[reoff[i]: reoff[i + 1]]])
                               for i in range(len(tl))])
        toff = synth.offsets(tl + gap)
        tp = np.empty(2 * len(tl) + 1, dtype=np.int64)
        tp[0] = 0
        tp[1::2] = toff[:-1] + gap
        tp[2::2] = toff[1:]
        out, ooff, st, err, olen = b64.decode_batch(to_dev(text), torch.from_numpy(tp).to(DEV))
        rout, rooff, rst, rerr, rolen = oracle.decode_batch(text, tp)
        assert np.array_equal(st.cpu().numpy(), rst)
        assert np.array_equal(err.cpu().numpy(), rerr)
        assert np.array_equal(olen.cpu().numpy(), rolen)
        o = out.cpu().numpy()
        for i in range(len(rolen)):
            assert np.array_equal(o[rooff[i]: rooff[i] + rolen[i]], rout[rooff[i]: rooff[i] + rolen[i]])


# ------------------------------------------------------------------ BASELINE.json configs at full size

def test_config1_full(b64):
    """1 MiB seed 0, std: encode 1,398,104 chars ('=='), round trip, 16 corruptions."""
    std = b64.standard()
    x = synth.data(1048576, seed=0)
    t = b64.encode(to_dev(x), std)
    ref = oracle.encode(x)
    assert t.numel() == 1398104 and np.array_equal(t.cpu().numpy(), ref)
    y, err = b64.decode(t, std)
    assert err == -1 and np.array_equal(y.cpu().numpy(), x)
    pos, bad = synth.corruption(16, ref.size, oracle.STANDARD, seed=0)
    t2 = ref.copy()
    t2[pos] = bad
    assert dec_check(b64, t2, oracle.STANDARD, oracle.PAD, std) == int(pos.min())


def test_config2_full(b64):
    """64 MiB at n, n+1, n+2 with std and url selected at runtime; full outputs vs oracle."""
    for n in (67108864, 67108865, 67108866):
        x = synth.data(n, seed=0)
        xd = to_dev(x)
        for chars, alpha in ((oracle.STANDARD, b64.standard()), (oracle.URL, b64.url())):
            t = b64.encode(xd, alpha)
            ref = oracle.encode(x, chars)
            assert t.numel() == 89478488
            assert np.array_equal(t.cpu().numpy(), ref)
            y, err = b64.decode(t, alpha)
            assert err == -1 and y.numel() == n and torch.equal(y, xd)


def test_config2_bench_step_grouped(b64):
    """configs[1] in bench.py's launch configurations: the 6 cases (n, n+1, n+2 x std, url) as
    ONE b64_decode_group launch + ONE b64_encode_group launch (the split step) and as ONE
    b64_codec_group launch (the headline step), + b64_decode_finalize_n; full outputs vs the
    oracle; three of the decode texts carry seeded corruptions."""
    cases = [(67108864 + d, chars, pad, alpha) for d in (0, 1, 2)
             for chars, pad, alpha in ((oracle.STANDARD, oracle.PAD, b64.standard()), (oracle.URL, oracle.PAD, b64.url()))]
    xs = [synth.data(n, seed=0) for n, *_ in cases]
    refs = [oracle.encode(x, chars, pad) for x, (n, chars, pad, _) in zip(xs, cases)]
    texts = []
    for i, r in enumerate(refs):
        t = r.copy()
        if i % 2 == 1:
            pos, bad = synth.corruption(3 + i, t.size, cases[i][1], seed=40 + i)
            t[pos] = bad
        texts.append(t)
    alph = [a for *_, a in cases]
    dxs, dts = [to_dev(x) for x in xs], [to_dev(t) for t in texts]
    douts, err, st = b64.decode_group(dts, alph)
    eouts = b64.encode_group(dxs, alph)
    errc, stc = err.cpu().numpy(), st.cpu().numpy()
    for i, (n, chars, pad, _) in enumerate(cases):
        assert np.array_equal(eouts[i].cpu().numpy(), refs[i]), i
        ref, rerr, rst = oracle.decode(texts[i], chars, pad)
        assert (errc[i], stc[i]) == (rerr, rst), i
        assert np.array_equal(douts[i][: ref.size].cpu().numpy(), ref), i
    # the bench's headline launches: the same 6 + 6 jobs as ONE b64_codec_group kernel, and as the
    # fused one (finalize in the kernel) twice in a row on the same error words
    results = [b64.codec_group(dxs, dts, alph, alph)]
    cells = torch.full((6,), b64.ERR_NONE, dtype=torch.int64, device=DEV)
    ticket = torch.zeros(1, dtype=torch.int32, device=DEV)
    for _ in range(2):
        results.append(b64.codec_group_fused(dxs, dts, alph, alph, cells=cells, ticket=ticket))
    for eouts, douts, err, st in results:
        errc, stc = err.cpu().numpy(), st.cpu().numpy()
        for i, (n, chars, pad, _) in enumerate(cases):
            assert np.array_equal(eouts[i].cpu().numpy(), refs[i]), i
            ref, rerr, rst = oracle.decode(texts[i], chars, pad)
            assert (errc[i], stc[i]) == (rerr, rst), i
            assert np.array_equal(douts[i][: ref.size].cpu().numpy(), ref), i


def _windows(total, count, width, seed):
    starts = (synth.words(seed, 7, 0, count) % np.uint64(max(total - width, 1))).astype(np.int64)
    return sorted(set([0, max(total - width, 0)] + starts.tolist()))


def test_config3_full_1gib(b64):
    """1 GiB encoded to 1,431,655,768 chars (device-generated); sampled windows vs oracle,
    round trip on device, and one corruption located exactly."""
    n = 1 << 30
    x = synth.device_data(n, seed=0)
    t = b64.encode(x)
    assert t.numel() == 1431655768
    for s in _windows(n // 3, 48, 4096, seed=3):
        a = 3 * s
        w = min(3 * 4096, n - a)
        ref = oracle.encode(synth.data(w, seed=0, offset=a))
        assert np.array_equal(t[4 * s: 4 * s + ref.size].cpu().numpy(), ref), s
    y, err = b64.decode(t)
    assert err == -1 and y.numel() == n and torch.equal(y, x)
    del y
    pos = 987_654_321
    t[pos] = ord("%")
    y, err = b64.decode(t)
    assert err == pos


def test_config4_full_batch(b64):
    """10^6 strings, log-uniform lengths in [1, 64 KiB]; sampled strings vs oracle, 1% corrupted."""
    count = 1_000_000
    L = synth.loguniform_lengths(count, seed=0)
    off = synth.offsets(L)
    total = int(off[-1])
    x = synth.device_data(total, seed=0)
    doff = torch.from_numpy(off).to(DEV)
    enc, eoff = b64.encode_batch(x, doff)
    reoff = np.zeros(count + 1, np.int64)
    np.cumsum(4 * ((L + 2) // 3), out=reoff[1:])
    assert np.array_equal(eoff.cpu().numpy(), reoff)
    sample = sorted(set((synth.words(0, 8, 0, 3000) % np.uint64(count)).astype(np.int64).tolist()) | {0, count - 1})
    for i in sample:
        xi = synth.data(int(L[i]), seed=0, offset=int(off[i]))
        assert np.array_equal(enc[reoff[i]: reoff[i + 1]].cpu().numpy(), oracle.encode(xi)), i
    picks = synth.pick(count, 0.01, seed=0)
    tl = np.diff(reoff)
    ppos = []
    for i in picks[:5000]:
        pos, bad = synth.corruption(1, int(tl[i]), oracle.STANDARD, seed=int(i))
        enc[int(reoff[i] + pos[0])] = int(bad[0])
        ppos.append(int(pos[0]))
    out, ooff, st, err, olen = b64.decode_batch(enc, eoff)
    stc, errc, olenc = st.cpu().numpy(), err.cpu().numpy(), olen.cpu().numpy()
    bad_idx = picks[:5000]
    assert np.array_equal(errc[bad_idx], np.array(ppos))
    assert (stc[bad_idx] == oracle.ST_BADCHAR).all()
    good = np.ones(count, bool)
    good[bad_idx] = False
    assert (errc[good] == -1).all() and (stc[good] == 0).all() and np.array_equal(olenc[good], L[good])
    oo = ooff.cpu().numpy()
    for i in sample:
        if good[i]:
            xi = synth.data(int(L[i]), seed=0, offset=int(off[i]))
            assert np.array_equal(out[oo[i]: oo[i] + L[i]].cpu().numpy(), xi), i


def test_config5_single_gpu_sampled(b64):
    """Config 5's 16 GiB stream on one GPU in 4 GiB shards (chunk API, aligned cuts),
    1000 corruptions, global err = min(positions); sampled windows vs oracle."""
    N = 1 << 34
    G = 4
    T = N // 3
    m = 4 * ((N + 2) // 3)
    pos, bad = synth.corruption(1000, m, oracle.STANDARD, seed=0)
    cells = torch.full((G,), b64.ERR_NONE, dtype=torch.int64, device=DEV)
    for r in range(G):
        t0 = (T * r // G) // 256 * 256
        t1 = (T * (r + 1) // G) // 256 * 256 if r < G - 1 else T
        a, b = 3 * t0, (3 * t1 if r < G - 1 else N)
        x = synth.device_data(b - a, seed=0, offset=a)
        t = b64.encode(x)
        for s in _windows((b - a) // 3, 6, 2048, seed=r):
            ref = oracle.encode(synth.data(min(3 * 2048, b - a - 3 * s), seed=0, offset=a + 3 * s))
            assert np.array_equal(t[4 * s: 4 * s + ref.size].cpu().numpy(), ref)
        c0, c1 = 4 * t0, 4 * t0 + t.numel()
        sel = (pos >= c0) & (pos < c1)
        if sel.any():
            t[torch.from_numpy(pos[sel] - c0).to(DEV)] = torch.from_numpy(bad[sel]).to(DEV)
        del x
        b64.decode_chunk(t, c0, r == G - 1, cells[r: r + 1])
        del t
        torch.cuda.empty_cache()
    eo = torch.empty(1, dtype=torch.int64, device=DEV)
    b64.decode_finalize(cells.min().reshape(1), eo)
    assert int(eo.item()) == int(pos.min())


def test_config5_bench_launch_sampled(b64):
    """configs[4] as bench.py times it on one GPU: the 16 GiB stream cut into the 8 shards an
    8-GPU run owns (dist rules), ONE encode_group launch and ONE decode_group launch over the
    8 shards with one shared error word; sampled text windows vs the oracle, 1000 injected
    errors, global first error, the exact output prefix before it."""
    from paper_1910_05109_b200 import dist as b64dist

    N, G = 1 << 34, 8
    x = synth.device_data(N, seed=0)
    m = b64.encoded_len(N)
    text = torch.empty(m, dtype=torch.uint8, device=DEV)
    es = [b64dist.encode_shard(N, G, r) for r in range(G)]
    b64.encode_group([x[sh.start: sh.stop] for sh in es],
                     outs=[text[sh.out_start: sh.out_start + (b64.encoded_len(sh.stop - sh.start) if sh.is_final
                                                              else 4 * ((sh.stop - sh.start) // 3))] for sh in es])
    for s0 in _windows(N // 3, 12, 2048, seed=5) + [es[3].start // 3 - 5, (N - 10) // 3]:
        ref = oracle.encode(synth.data(min(3 * 2048, N - 3 * s0), seed=0, offset=3 * s0))
        assert np.array_equal(text[4 * s0: 4 * s0 + ref.size].cpu().numpy(), ref), s0
    pos, bad = synth.corruption(1000, m, oracle.STANDARD, seed=0)
    text[torch.from_numpy(pos).to(DEV)] = torch.from_numpy(bad).to(DEV)
    del x
    torch.cuda.empty_cache()
    out = torch.empty(3 * (m // 4), dtype=torch.uint8, device=DEV)
    ds = [b64dist.decode_shard(m, G, r) for r in range(G)]
    cell = torch.full((1,), b64.ERR_NONE, dtype=torch.int64, device=DEV)
    items = (b64._lib.DecodeItem * G)()
    std = b64.standard()
    for r, sh in enumerate(ds):
        t_r = text[sh.start: sh.stop]
        o_r = out[sh.out_start: sh.out_start + 3 * ((sh.stop - sh.start) // 4)]
        items[r] = b64._lib.DecodeItem(t_r.data_ptr(), t_r.numel(), o_r.data_ptr(), ctypes.pointer(std), sh.start,
                                       int(sh.is_final), 0, cell.data_ptr())
    b64._lib.check(b64._lib.lib().b64_decode_group(items, G, None), "b64_decode_group")
    eo = torch.empty(1, dtype=torch.int64, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    b64.decode_finalize(cell, eo, st)
    first = int(pos.min())
    assert (int(eo.item()), int(st.item())) == (first, oracle.ST_BADCHAR)
    k = 3 * (first // 4)
    assert np.array_equal(out[:k].cpu().numpy(), synth.data(k, seed=0))
    del text, out
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ host-buffer pipeline

def test_host_pipeline_vs_oracle(b64):
    """b64_encode_host / b64_decode_host with small chunks (many rotations of the 3 buffers)."""
    pipe = b64.HostPipeline(chunk_bytes=3072 * 5)
    for n in (0, 1, 2, 3, 3071, 3072, 3073, 15360 * 3 + 5, 200_003):
        for chars, alpha in ((oracle.STANDARD, b64.standard()), (oracle.URL, b64.url())):
            x = synth.data(n, seed=n + 1)
            xh = torch.from_numpy(x).pin_memory()
            t = pipe.encode(xh, alpha)
            ref = oracle.encode(x, chars)
            assert np.array_equal(t.numpy(), ref), n
            y, err = pipe.decode(t.clone().pin_memory(), alpha)
            assert err == -1 and np.array_equal(y.numpy(), x), n
            if ref.size > 8:
                pos, bad = synth.corruption(3, ref.size, chars, seed=n)
                t2 = ref.copy()
                t2[pos] = bad
                y, err = pipe.decode(torch.from_numpy(t2).pin_memory(), alpha)
                rref, rerr, rst = oracle.decode(t2, chars)
                assert err == rerr == int(pos.min())
                assert np.array_equal(y.numpy(), rref)


def test_host_pipeline_overlapped_calls(b64):
    """Back-to-back sync=False host calls (two workspaces, B64_HOST_CALLER_ORDERED): calls
    overlap each other; every output and error word must still match the oracle."""
    pipe = b64.HostPipeline(chunk_bytes=3072 * 7)
    jobs = []
    for i, n in enumerate((100_003, 5, 3072 * 7 * 3 + 11, 64_000, 0, 250_001, 3)):
        chars, alpha = ((oracle.STANDARD, b64.standard()), (oracle.URL, b64.url()))[i % 2]
        x = synth.data(n, seed=700 + i)
        ref = oracle.encode(x, chars)
        t2 = ref.copy()
        if ref.size > 8 and i % 2 == 0:
            pos, bad = synth.corruption(2, ref.size, chars, seed=i)
            t2[pos] = bad
        xh = torch.from_numpy(x).pin_memory()
        th = torch.from_numpy(t2).pin_memory()
        eo = torch.empty(max(ref.size, 1), dtype=torch.uint8).pin_memory()
        do = torch.empty(max(3 * (ref.size // 4), 1), dtype=torch.uint8).pin_memory()
        jobs.append((chars, x, ref, t2, xh, th, eo, do, alpha))
    results = []
    for rep in range(2):
        for chars, x, ref, t2, xh, th, eo, do, alpha in jobs:
            te = pipe.encode(xh, alpha, out=eo, sync=False)
            yo, info = pipe.decode(th, alpha, out=do, sync=False)
            results.append((te, yo, info))
    pipe.join()
    torch.cuda.synchronize()
    for k, (te, yo, info) in enumerate(results):
        chars, x, ref, t2, *_ = jobs[k % len(jobs)]
        assert np.array_equal(te.numpy()[: ref.size], ref), k
        rref, rerr, rst = oracle.decode(t2, chars)
        err, st = int(info[0].item()), int(info[1:2].view(torch.int32)[0].item())
        assert (err, st) == (rerr, rst), k
        assert np.array_equal(yo.numpy()[: rref.size], rref), k


# ------------------------------------------------------------------ guard bands (no writes outside the output)

def test_no_writes_outside_outputs(b64):
    """Canary bytes around (and, for decode, after out_len inside) every output buffer stay intact:
    fast and generic kernels, single stream and batch."""
    G = 256
    for n in (1, 2, 3, 100, 767, 768, 769, 4096 * 3 + 1, 300_001):
        for oi, oo in ((0, 0), (1, 3), (5, 16), (0, 7)):
            x = synth.data(n, seed=n)
            m = b64.encoded_len(n)
            buf = torch.full((m + 2 * G + 32,), 0xA5, dtype=torch.uint8, device=DEV)
            dst = buf[G + oo: G + oo + m]
            b64.encode(to_dev(x, oi), out=dst)
            hb = buf.cpu().numpy()
            assert (hb[: G + oo] == 0xA5).all() and (hb[G + oo + m:] == 0xA5).all(), (n, oi, oo)
            text = oracle.encode(x)
            cap = 3 * (m // 4)
            buf = torch.full((cap + 2 * G + 32,), 0xA5, dtype=torch.uint8, device=DEV)
            dst = buf[G + oo: G + oo + cap]
            out, info = b64.decode_async(to_dev(text, oi), out=dst)
            err, st, olen = info.tolist()
            assert err == -1 and olen == n
            hb = buf.cpu().numpy()
            assert (hb[: G + oo] == 0xA5).all() and (hb[G + oo + n:] == 0xA5).all(), (n, oi, oo)
    # batch: outputs land exactly in their slots; gaps left between slots stay intact
    L = synth.loguniform_lengths(2000, hi=3000, seed=9)
    off = synth.offsets(L)
    x = synth.data(int(off[-1]), seed=9)
    el = 4 * ((L + 2) // 3)
    eoff = np.zeros(L.size + 1, np.int64)
    np.cumsum(el + 8, out=eoff[1:])  # 8 canary bytes after every string's slot
    buf = torch.full((int(eoff[-1]) + 64,), 0xA5, dtype=torch.uint8, device=DEV)
    b64.encode_batch(to_dev(x), torch.from_numpy(off).to(DEV), out=buf, out_off=torch.from_numpy(eoff).to(DEV))
    hb = buf.cpu().numpy()
    for i in range(L.size):
        assert (hb[eoff[i] + el[i]: eoff[i + 1]] == 0xA5).all(), i


def test_dist_layer_world1_cuda(b64):
    """dist.encode_sharded / decode_sharded with the CUDA codec and no process group (world 1)."""
    from paper_1910_05109_b200 import dist as b64dist

    x = synth.data(768 * 40 + 2, seed=77)
    sh = b64dist.encode_shard(x.size, 1, 0)
    t = b64dist.encode_sharded(to_dev(x))
    ref = oracle.encode(x)
    assert sh.is_final and np.array_equal(t.cpu().numpy(), ref)
    t2 = ref.copy()
    t2[5000] = ord("~")
    ds = b64dist.decode_shard(t2.size, 1, 0)
    out, err, st = b64dist.decode_sharded(to_dev(t2), ds)
    assert (err, st) == (5000, oracle.ST_BADCHAR)
    assert np.array_equal(out[: 3 * (5000 // 4)].cpu().numpy(), x[: 3 * (5000 // 4)])


# ------------------------------------------------------------------ grouped launches

def test_group_encode_decode_vs_oracle(b64):
    al = _alphabets(b64)
    sizes = [0, 1, 2, 3, 767, 768, 769, 5000, 100_003, 768 * 300 + 1, 768 * 1000 + 2, 64, 3 * 1024]
    for rep in range(2):
        xs, refs, chars_l, alph_l, offs = [], [], [], [], []
        for i, n in enumerate(sizes):
            chars, pad, alpha = al[(i + rep) % len(al)]
            x = synth.data(n, seed=1000 * rep + i)
            xs.append(x)
            refs.append(oracle.encode(x, chars, pad))
            chars_l.append((chars, pad))
            alph_l.append(alpha)
        # some items misaligned (own launch), others grouped (more than 8 -> two groups)
        dx = [to_dev(x, 1 if (i % 5 == 4) else 0) for i, x in enumerate(xs)]
        outs = b64.encode_group(dx, alph_l)
        for i in range(len(sizes)):
            assert np.array_equal(outs[i].cpu().numpy(), refs[i]), (rep, i)
        texts = []
        for i, r in enumerate(refs):
            t = r.copy()
            if i % 3 == 1 and t.size > 4:
                pos, bad = synth.corruption(2, t.size, chars_l[i][0], seed=i, pad=chars_l[i][1])
                t[pos] = bad
            texts.append(t)
        dt = [to_dev(t, 3 if (i % 4 == 3) else 0) for i, t in enumerate(texts)]
        douts, err, st = b64.decode_group(dt, alph_l)
        errc, stc = err.cpu().numpy(), st.cpu().numpy()
        for i, t in enumerate(texts):
            ref, rerr, rst = oracle.decode(t, *chars_l[i])
            assert (errc[i], stc[i]) == (rerr, rst), (rep, i)
            assert np.array_equal(douts[i][: ref.size].cpu().numpy(), ref), (rep, i)


def test_group_unequal_large_streams(b64):
    """Warp-partitioned groups: streams of very different chunk counts (many warps per
    large stream, one warp for a tiny one, none for an empty one) vs the oracle."""
    al = _alphabets(b64)
    sizes = [40 << 20, (3 << 20) + 5, 1024, 0, (17 << 20) + 2, 768 * 7]
    xs = [synth.data(n, seed=500 + i) for i, n in enumerate(sizes)]
    chars_l = [(al[i % len(al)][0], al[i % len(al)][1]) for i in range(len(sizes))]
    alph_l = [al[i % len(al)][2] for i in range(len(sizes))]
    outs = b64.encode_group([to_dev(x) for x in xs], alph_l)
    texts = []
    for i, x in enumerate(xs):
        ref = oracle.encode(x, *chars_l[i])
        assert np.array_equal(outs[i].cpu().numpy(), ref), i
        t = ref.copy()
        if i in (0, 4) and t.size > 4:
            pos, bad = synth.corruption(3, t.size, chars_l[i][0], seed=i, pad=chars_l[i][1])
            t[pos] = bad
        texts.append(t)
    douts, err, st = b64.decode_group([to_dev(t) for t in texts], alph_l)
    errc, stc = err.cpu().numpy(), st.cpu().numpy()
    for i, t in enumerate(texts):
        ref, rerr, rst = oracle.decode(t, *chars_l[i])
        assert (errc[i], stc[i]) == (rerr, rst), i
        k = ref.size if rerr < 0 else 3 * (rerr // 4)
        assert np.array_equal(douts[i][:k].cpu().numpy(), ref[:k]), i


def test_codec_group_mixed(b64):
    """b64_codec_group: encodes and decodes in ONE launch (decode CTAs + encode CTAs), unequal
    sizes, corrupted texts, several groups (> 8 + 8 items), misaligned items in between."""
    al = _alphabets(b64)
    rng = np.random.default_rng(12)
    sizes = [40 << 20, 5, (3 << 20) + 1, 0, 768 * 9 + 2] + [int(v) for v in rng.integers(0, 400_000, 14)]
    xs = [synth.data(n, seed=950 + i) for i, n in enumerate(sizes)]
    chars_l = [al[i % len(al)][:2] for i in range(len(sizes))]
    alph_l = [al[i % len(al)][2] for i in range(len(sizes))]
    texts = [oracle.encode(x, *chars_l[i]) for i, x in enumerate(xs)]
    for i in range(0, len(texts), 3):
        if texts[i].size > 8:
            pos, bad = synth.corruption(2, texts[i].size, chars_l[i][0], seed=i, pad=chars_l[i][1])
            texts[i][pos] = bad
    dx = [to_dev(x, 1 if i % 7 == 6 else 0) for i, x in enumerate(xs)]
    order = list(range(len(texts)))[::-1]  # decode list in another order than the encode list
    dt = [to_dev(texts[i], 2 if i % 6 == 5 else 0) for i in order]
    eouts, douts, err, st = b64.codec_group(dx, dt, alph_l, [alph_l[i] for i in order])
    errc, stc = err.cpu().numpy(), st.cpu().numpy()
    for i, x in enumerate(xs):
        assert np.array_equal(eouts[i].cpu().numpy(), oracle.encode(x, *chars_l[i])), i
    for j, i in enumerate(order):
        ref, rerr, rst = oracle.decode(texts[i], *chars_l[i])
        assert (errc[j], stc[j]) == (rerr, rst), i
        k = ref.size if rerr < 0 else 3 * (rerr // 4)
        assert np.array_equal(douts[j][:k].cpu().numpy(), ref[:k]), i
    # one kind only
    eouts, douts, err, st = b64.codec_group(dx[:3], [], alph_l[:3])
    assert douts == [] and err is None
    for i in range(3):
        assert np.array_equal(eouts[i].cpu().numpy(), oracle.encode(xs[i], *chars_l[i])), i


def test_codec_group_fused(b64):
    """b64_codec_group_fused: ONE launch whose last CTA finalises and resets the error words and
    the ticket; back-to-back calls with the same cells / ticket and changing corruptions, empty
    items, a decode-only and an encode-only call, and the refusal of non-fusable lists."""
    al = _alphabets(b64)
    sizes = [3 << 20, 768 * 5 + 1, 0, 100_003, (1 << 20) + 2]
    xs = [synth.data(n, seed=60 + i) for i, n in enumerate(sizes)]
    chars_l = [al[i % len(al)][:2] for i in range(len(sizes))]
    alph_l = [al[i % len(al)][2] for i in range(len(sizes))]
    refs = [oracle.encode(x, *chars_l[i]) for i, x in enumerate(xs)]
    dx = [to_dev(x) for x in xs]
    cells = torch.full((len(sizes),), b64.ERR_NONE, dtype=torch.int64, device=DEV)
    ticket = torch.zeros(1, dtype=torch.int32, device=DEV)
    for rep in range(4):
        texts = []
        for i, r in enumerate(refs):
            t = r.copy()
            if (i + rep) % 2 and t.size > 4:
                pos, bad = synth.corruption(1 + rep, t.size, chars_l[i][0], seed=10 * rep + i, pad=chars_l[i][1])
                t[pos] = bad
            texts.append(t)
        dt = [to_dev(t) for t in texts]
        eouts, douts, err, st = b64.codec_group_fused(dx, dt, alph_l, alph_l, cells=cells, ticket=ticket)
        errc, stc = err.cpu().numpy(), st.cpu().numpy()
        for i in range(len(sizes)):
            assert np.array_equal(eouts[i].cpu().numpy(), refs[i]), (rep, i)
            ref, rerr, rst = oracle.decode(texts[i], *chars_l[i])
            assert (errc[i], stc[i]) == (rerr, rst), (rep, i)
            k = ref.size if rerr < 0 else 3 * (rerr // 4)
            assert np.array_equal(douts[i][:k].cpu().numpy(), ref[:k]), (rep, i)
        # the kernel left the words and the ticket ready for the next call
        assert torch.all(cells == b64.ERR_NONE) and int(ticket.item()) == 0
    _, douts, err, st = b64.codec_group_fused([], [to_dev(refs[0])], dec_alphabets=alph_l[0], cells=cells[:1],
                                              ticket=ticket)
    assert int(err.item()) == -1 and torch.equal(douts[0][: xs[0].size], dx[0])
    eouts, _, _, _ = b64.codec_group_fused(dx[:2], [], alph_l[:2], ticket=ticket)
    assert np.array_equal(eouts[1].cpu().numpy(), refs[1]) and int(ticket.item()) == 0
    with pytest.raises(b64.B64Error, match="EINVAL"):  # misaligned item: not fusable
        b64.codec_group_fused([to_dev(xs[1], 1)], [], alph_l[1], ticket=ticket)
    with pytest.raises(b64.B64Error, match="EINVAL"):  # more than 8 items
        b64.codec_group_fused(dx[1:2] * 9, [], alph_l[1], ticket=ticket)


def test_group_decode_as_shards(b64):
    """Grouped items as shards of one stream: global bases, only the last is final, one cell."""
    x = synth.data(768 * 500 + 1, seed=3)
    text = oracle.encode(x)
    for trial in range(4):
        t2 = text.copy()
        if trial:
            pos, bad = synth.corruption(trial, text.size, oracle.STANDARD, seed=trial)
            t2[pos] = bad
        ref, rerr, rst = oracle.decode(t2)
        cuts = [0, 1024 * 100, 1024 * 101, 1024 * 350, t2.size]
        dt = to_dev(t2)
        parts = [dt[cuts[i]: cuts[i + 1]] for i in range(len(cuts) - 1)]
        cell = torch.full((1,), b64.ERR_NONE, dtype=torch.int64, device=DEV)
        items = (b64._lib.DecodeItem * len(parts))()
        outs = [torch.empty(3 * (p.numel() // 4), dtype=torch.uint8, device=DEV) for p in parts]
        std = b64.standard()
        for i, p in enumerate(parts):
            items[i] = b64._lib.DecodeItem(p.data_ptr(), p.numel(), outs[i].data_ptr(), ctypes.pointer(std),
                                           cuts[i], int(i == len(parts) - 1), 0, cell.data_ptr())
        b64._lib.check(b64._lib.lib().b64_decode_group(items, len(parts), None), "group")
        eo = torch.empty(1, dtype=torch.int64, device=DEV)
        b64.decode_finalize(cell, eo)
        assert int(eo.item()) == rerr
        got = torch.cat(outs).cpu().numpy()
        assert np.array_equal(got[: ref.size], ref)


def test_decode_fast_path_small_sizes(b64):
    """b64_decode_ex takes the single-launch cluster kernel up to 512 Ki chars; the multi-CTA
    bulk kernel (b64_decode_chunk + finalize) must agree with the oracle on the same sizes."""
    std = b64.standard()
    for n in (0, 1, 2, 3, 767, 768, 3 * 1024 + 2, 100_001, 768 * 300 + 1, 3_000_000, 3_200_000):
        x = synth.data(n, seed=n + 5)
        text = oracle.encode(x)
        for trial in range(3):
            t2 = text.copy()
            if trial and t2.size:
                pos, bad = synth.corruption(trial, t2.size, oracle.STANDARD, seed=n + trial)
                t2[pos] = bad
            ref, rerr, rst = oracle.decode(t2)
            dt = to_dev(t2)
            cell = torch.full((1,), b64.ERR_NONE, dtype=torch.int64, device=DEV)
            out = b64.decode_chunk(dt, 0, True, cell, std)
            eo = torch.empty(1, dtype=torch.int64, device=DEV)
            st = torch.zeros(1, dtype=torch.int32, device=DEV)
            b64.decode_finalize(cell, eo, st)
            assert (int(eo.item()), int(st.item())) == (rerr, rst), (n, trial)
            assert np.array_equal(out[: ref.size].cpu().numpy(), ref)
            assert dec_check(b64, t2, oracle.STANDARD, oracle.PAD, std) == rerr  # small cluster path


def test_decode_ex_small_path_many_ctas(b64):
    """Around the cluster-size and kSmallMax boundaries (16 CTAs x 16 warps x 1024 chars; 512 Ki chars),
    errors at the start, middle and in the final quad (the prefetched chunk loop and its tail)."""
    std = b64.standard()
    for m_chars in (16 * 1024 - 4, 16 * 1024, 256 * 1024, 256 * 1024 + 4096, (512 << 10) - 4, 512 << 10,
                    (512 << 10) + 4, (1536 << 10) - 4, 1536 << 10, (1536 << 10) + 4, 4 << 20):
        n = m_chars // 4 * 3 - 1
        x = synth.data(n, seed=m_chars)
        text = oracle.encode(x)
        dec_check(b64, text, oracle.STANDARD, oracle.PAD, std)
        for p in (0, text.size // 2, text.size - 3, text.size - 1):
            t2 = text.copy()
            t2[p] = ord("#")
            dec_check(b64, t2, oracle.STANDARD, oracle.PAD, std)


# ------------------------------------------------------------------ padding-optional decode (R13)

def test_decode_unpadded_vs_oracle(b64):
    al = _alphabets(b64)
    for n in list(range(0, 200)) + [767, 768, 769, 3 * 1024 + 1, 100_001, 1 << 20, (1 << 20) + 1, 3_000_001]:
        chars, pad, alpha = al[n % len(al)]
        x = synth.data(n, seed=n + 9)
        bare = oracle.encode_unpadded(x, chars, pad)
        variants = [bare, oracle.encode(x, chars, pad)]
        if bare.size:
            t2 = bare.copy()
            pos, bad = synth.corruption(1 + n % 2, t2.size, chars, seed=n, pad=pad)
            t2[pos] = bad
            variants.append(t2)
            t3 = bare.copy()
            t3[-1] = pad  # '=' inside a partial group is a bad char
            variants.append(t3)
            if bare.size % 4 in (2, 3):
                t4 = bare.copy()
                t4[-1] = chars[(chars.index(bytes([t4[-1]])) + 1) % 64]  # dirty dropped bits
                variants.append(t4)
        for t in variants:
            if t.size % 4 == 1:
                with pytest.raises(b64.B64Error, match="ELENGTH"):
                    b64.decode_unpadded(to_dev(t), alpha)
                continue
            ref, rerr, rst = oracle.decode_unpadded(t, chars, pad)
            out, err = b64.decode_unpadded(to_dev(t), alpha)
            assert err == rerr, (n, err, rerr)
            assert np.array_equal(out.cpu().numpy(), ref), n


# ------------------------------------------------------------------ whitespace-skipping decode (R14)

_WS = np.frombuffer(b" \t\n\r\x0b\x0c", np.uint8)


def _mime(text: np.ndarray, seed: int, every: int = 76, extra: int = 0) -> np.ndarray:
    """CRLF after every `every` chars plus `extra` random whitespace bytes at seeded positions."""
    parts = []
    for i in range(0, text.size, every):
        parts.append(text[i: i + every])
        parts.append(np.frombuffer(b"\r\n", np.uint8))
    out = np.concatenate(parts) if parts else text.copy()
    if extra:
        w = synth.words(seed, 13, 0, 2 * extra)
        pos = np.sort((w[:extra] % np.uint64(out.size + 1)).astype(np.int64))
        vals = _WS[(w[extra:] % np.uint64(_WS.size)).astype(np.int64)]
        out = np.insert(out, pos, vals)
    return out


def test_decode_ws_vs_oracle(b64):
    al = _alphabets(b64)
    ws_alpha = oracle.STANDARD[:62] + b" \t"  # whitespace chars that are data
    cases = []
    for n in (0, 1, 2, 3, 57, 100, 3000, 4096 * 3 + 5, 100_001, 1_000_003, 6_000_000):
        cases.append(n)
    for i, n in enumerate(cases):
        chars, pad, alpha = al[i % len(al)]
        x = synth.data(n, seed=n + 21)
        text = oracle.encode(x, chars, pad)
        variants = [_mime(text, n, every=76, extra=3), _mime(text, n, every=1 + n % 97, extra=50)]
        if text.size > 8:
            t2 = _mime(text, n + 1, every=64, extra=5)
            keep = np.nonzero(~np.isin(t2, _WS))[0]
            p = int(keep[int(synth.words(n, 14, 0, 1)[0] % max(keep.size - 4, 1))])
            t2 = t2.copy()
            t2[p] = ord("*")
            variants.append(t2)
            t3 = _mime(text[:-1], n + 2, every=50, extra=2)  # compacted length % 4 != 0
            variants.append(t3)
        variants.append(np.frombuffer(b"\r\n \t" * 9, np.uint8).copy())
        for t in variants:
            ref, rerr, rst = oracle.decode_ws(t, chars, pad)
            out, err = b64.decode_ws(to_dev(t), alpha)
            assert err == rerr, (n, err, rerr, rst)
            assert np.array_equal(out.cpu().numpy(), ref), n
    # whitespace that belongs to the alphabet is data
    _decode_ws_adversarial(b64)
    a2 = b64.alphabet(ws_alpha)
    x = synth.data(5000, seed=4)
    t = oracle.encode(x, ws_alpha)
    out, err = b64.decode_ws(to_dev(_mime(t, 4, every=33)), a2)
    ref, rerr, _ = oracle.decode_ws(_mime(t, 4, every=33), ws_alpha)
    assert err == rerr and np.array_equal(out.cpu().numpy(), ref)


def test_decode_fused_ctx(b64):
    """b64_decode_fused (one launch, self-resetting DecodeContext) equals b64_decode_ex / the oracle
    -- err_off, status, out_len, bytes -- call after call on the same context with valid and
    corrupted texts (interior and final-quad errors), strict and lenient alphabets, sizes below
    and above the cluster threshold, unaligned buffers (3-op path), and replayed from a graph."""
    al = _alphabets(b64)
    ctx = b64.DecodeContext()
    rng = np.random.default_rng(31)
    for trial, n in enumerate([0, 1, 5, 400_000, 1 << 20, (1 << 20) + 1, 3_000_002, 25_000_001]):
        chars, pad, alpha = al[trial % len(al)]
        ref_t = oracle.encode(synth.data(n, seed=500 + trial), chars, pad)
        for rep in range(4):
            text = ref_t.copy()
            if rep % 2 and text.size:
                k = int(rng.integers(1, 4))
                pos, bad = synth.corruption(k, text.size, chars, seed=trial * 10 + rep, pad=pad)
                text[pos] = bad
            if rep == 3 and text.size >= 4 and ref_t[-1] == pad:
                text[-2] = chars[1]  # 'x?b=' or 'xb==' -> a final-quad error of some kind
            for lenient in (False, True):
                a = b64.lenient_of(alpha) if lenient else alpha
                ref, rerr, rst = oracle.decode(text, chars, pad, lenient=lenient)
                out, info = b64.decode_async(to_dev(text), a, ctx=ctx)
                err, stt, olen = info.tolist()
                assert (err, stt) == (rerr, rst), (n, rep, lenient, err, stt, rerr, rst)
                assert olen == (ref.size if rerr < 0 else 3 * (rerr // 4)), (n, rep, olen)
                assert np.array_equal(out[:olen].cpu().numpy(), ref[:olen]), (n, rep)
        # unaligned input: falls back to the 3-op path, same results
        out, err = b64.decode(to_dev(ref_t, 1), alpha, ctx=ctx)
        assert err == -1 and out.numel() == b64.decoded_len_max(ref_t.size) - int(np.sum(ref_t[-2:] == pad))
    # graph replay of a fused decode: every replay gives the result
    x = synth.data(3_000_000, seed=9)
    t = to_dev(oracle.encode(x))
    info = b64.new_info()
    o = torch.empty(b64.decoded_len_max(t.numel()), dtype=torch.uint8, device=DEV)
    g, sg = torch.cuda.CUDAGraph(), torch.cuda.Stream()
    sg.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(sg):
        gctx = b64.DecodeContext(stream=sg)
        b64.decode_async(t, out=o, info=info, ctx=gctx)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=sg):
            for _ in range(3):
                b64.decode_async(t, out=o, info=info, ctx=gctx)
    torch.cuda.current_stream().wait_stream(sg)
    for _ in range(3):
        info.zero_()
        o.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert info.tolist() == [-1, 0, x.size] and np.array_equal(o[: x.size].cpu().numpy(), x)


def test_concurrent_streams_and_contexts(b64):
    """Decodes (fused single-launch with one context per stream, plain, MIME) and encodes issued
    on 4 streams at once, twice over, with no host sync in between: every result equals the
    oracle's (contexts and workspaces are per call / per stream; the library keeps no per-call
    state)."""
    streams = [torch.cuda.Stream() for _ in range(4)]
    ctxs = [b64.DecodeContext(stream=s_) for s_ in streams]
    torch.cuda.synchronize()
    data = [synth.data(n, seed=40 + i) for i, n in enumerate((2_000_003, 700_001, 5_000_000, 1_500_002))]
    texts = [oracle.encode(x) for x in data]
    bad = [t.copy() for t in texts]
    for i, t in enumerate(bad):
        t[(i + 1) * 10_007] = ord("*")
    dts, dbad = [to_dev(t) for t in texts], [to_dev(t) for t in bad]
    dxs = [to_dev(x) for x in data]
    res = []
    for rep in range(2):
        for i, s_ in enumerate(streams):
            with torch.cuda.stream(s_):
                src = dbad[i] if (i + rep) % 2 else dts[i]
                res.append((i, rep, b64.decode_async(src, ctx=ctxs[i]), b64.decode_async(src),
                            b64.encode(dxs[i])))
    torch.cuda.synchronize()
    for i, rep, (o1, inf1), (o2, inf2), e in res:
        t = bad[i] if (i + rep) % 2 else texts[i]
        ref, rerr, rst = oracle.decode(t)
        for o, inf in ((o1, inf1), (o2, inf2)):
            err, stt, olen = inf.tolist()
            assert (err, stt) == (rerr, rst), (i, rep, err, rerr)
            k = ref.size if rerr < 0 else 3 * (rerr // 4)
            assert olen == k and np.array_equal(o[:k].cpu().numpy(), ref[:k]), (i, rep)
        assert np.array_equal(e.cpu().numpy(), texts[i]), (i, rep)


def test_decode_ws_small_single_launch(b64):
    """Texts up to the single-launch size (one cluster: 1-16 CTAs of 16 warps, 8 KiB per CTA step):
    sizes around the CTA and warp-slice boundaries, random whitespace, an error in every CTA's
    slice in turn, the LENGTH rule, all-whitespace text, unaligned input, lenient alphabet --
    bytes, err_off (original coordinates) and status equal the oracle's."""
    rng = np.random.default_rng(17)
    ws = np.frombuffer(b" \t\n\r\x0b\x0c", np.uint8)
    for target in (5, 511, 512, 513, 8191, 8192, 8193, 3 * 8192 + 7, 100_000, 400_000, 524_288):
        n = max(1, (target * 3) // 4 - target // 40)
        t = oracle.encode(synth.data(n, seed=target))
        k = max(0, target - t.size)
        pos = np.sort(rng.integers(0, t.size + 1, k))
        text = np.insert(t, pos, ws[rng.integers(0, 6, k)])[:target] if k else t[:target]
        variants = [text]
        R = min(16, max(1, (text.size + 8191) // 8192))
        C = (((text.size + R - 1) // R) + 8191) // 8192 * 8192
        for r in range(R):  # one bad char in each CTA's slice
            keep = np.nonzero(~np.isin(text, ws))[0]
            cand = keep[(keep >= r * C) & (keep < (r + 1) * C)]
            if cand.size:
                v = text.copy()
                v[cand[cand.size // 2]] = ord("*")
                variants.append(v)
        variants.append(np.concatenate([text, np.frombuffer(b"A", np.uint8)]))  # kept % 4 != 0 (usually)
        variants.append(np.full(min(target, 3000), ord(" "), np.uint8))          # whitespace only
        for i, v in enumerate(variants):
            for lenient in (False, True):
                ref, rerr, rst = oracle.decode_ws(v, lenient=lenient)
                a = b64.lenient_of(b64.standard()) if lenient else b64.standard()
                out, err = b64.decode_ws(to_dev(v, i % 2), a)
                assert err == rerr, (target, i, lenient, err, rerr, rst)
                assert np.array_equal(out.cpu().numpy(), ref), (target, i, lenient)


def test_decode_ws_line_structured(b64):
    """MIME / PEM line layouts (the one-pass line path of b64_decode_ws) and their near misses
    (which take the general path): every result equals the oracle's -- bytes, err_off in the
    ORIGINAL text, status."""
    def lines(t, L, sep=b"\r\n", trail=True):
        parts = []
        for i in range(0, t.size, L):
            parts.append(t[i: i + L])
            if trail or i + L < t.size:
                parts.append(np.frombuffer(sep, np.uint8))
        return np.concatenate(parts) if parts else t.copy()

    al = _alphabets(b64)
    cases = []
    for n in (1, 2, 3, 54, 57, 58, 1000, 4096 * 3 + 1, 100_000, 1_000_002):
        for L, sep, trail in ((76, b"\r\n", True), (76, b"\r\n", False), (64, b"\n", True), (64, b"\n", False),
                              (4, b"\r\n", True), (72, b" ", False)):
            t = oracle.encode(synth.data(n, seed=n + L))
            cases.append(lines(t, L, sep, trail))
    t = oracle.encode(synth.data(100_000, seed=5))
    mime = lines(t, 76)
    k = mime.size // 2
    variants = []
    for pos, val in ((k, ord("*")), (k, ord("=")), (77, ord("A")), (76, ord("A")), (78 * 5 + 3, ord("\n")),
                     (mime.size - 3, ord("A")), (mime.size - 4, ord("A")), (mime.size - 1, ord("x"))):
        v = mime.copy()
        v[pos] = val
        variants.append(v)  # bad char / '=' / a separator byte replaced / a whitespace byte inside a line
    variants.append(np.concatenate([mime, np.frombuffer(b"\r\n", np.uint8)]))      # a blank line at the end
    variants.append(np.concatenate([mime, np.frombuffer(b"\r\n\r\n  \t\n", np.uint8)]))  # trailing blanks
    variants.append(np.concatenate([mime[:-2], np.full(70_000, ord(" "), np.uint8)]))  # past the probe window
    variants.append(np.concatenate([lines(t, 76, trail=False), np.frombuffer(b"   ", np.uint8)]))
    variants.append(np.concatenate([np.frombuffer(b"\r\n \t", np.uint8), mime]))          # leading blanks
    variants.append(np.concatenate([np.full(70_001, ord("\n"), np.uint8), mime]))        # past the probe window
    v = np.concatenate([np.frombuffer(b"\n\n", np.uint8), mime]).copy()
    v[2 + 78 * 3 + 10] = ord("*")                                                      # offset + bad char
    variants.append(v)
    variants.append(lines(t, 75))                                                   # L % 4 != 0
    variants.append(np.concatenate([lines(t[:7600], 76), lines(t[7600:], 64)]))    # line length changes
    variants.append(lines(t[:-1], 76))                                              # kept chars % 4 != 0
    variants.append(lines(t[:-3], 76, trail=False))
    variants.append(np.frombuffer(b"\r\n", np.uint8).copy())
    variants.append(lines(oracle.encode(synth.data(57, seed=1)), 76)[:-1])           # separator cut short
    for i, c in enumerate(cases + variants):
        chars, pad, alpha = al[i % len(al)] if i < len(cases) else al[0]
        if i < len(cases) and (chars, pad) != (oracle.STANDARD, oracle.PAD):
            c = oracle.encode(oracle.decode_ws(c)[0], chars, pad)  # re-encode in this alphabet, same layout
            c = lines(c, [76, 76, 64, 64, 4, 72][i % 6], [b"\r\n", b"\r\n", b"\n", b"\n", b"\r\n", b" "][i % 6],
                      [True, False, True, False, True, False][i % 6])
        for lenient in (False, True):
            ref, rerr, rst = oracle.decode_ws(c, chars, pad, lenient=lenient)
            a = b64.lenient_of(alpha) if lenient else alpha
            out, err = b64.decode_ws(to_dev(c, i % 3), a)
            assert err == rerr, (i, lenient, err, rerr, rst)
            assert np.array_equal(out.cpu().numpy(), ref), (i, lenient)


def _decode_ws_adversarial(b64):
    """Whitespace layouts around the 4 KiB chunks of the fused decode: long runs spanning
    chunks, chunks holding 0-3 kept chars, quads (and the final quad) split across chunks by
    whitespace, errors in the look-ahead chars and in a split final quad, '=' misplaced,
    unaligned input (byte path), lenient alphabet."""
    x = synth.data(30_000, seed=91)
    text = oracle.encode(x)  # 40000 chars, no padding
    xp = synth.data(30_001, seed=92)
    textp = oracle.encode(xp)  # ends 'xx=='
    sp = lambda k: np.full(k, ord(" "), np.uint8)  # noqa: E731
    cat = lambda *a: np.concatenate(a)  # noqa: E731
    cases = [
        cat(text[:5000], sp(10_000), text[5000:]),                          # run over 2+ chunks
        cat(*[cat(text[i: i + 1], sp(1500)) for i in range(12)], text[12:]),  # chunks with 1-3 kept chars
        cat(textp[:-2], sp(5000), textp[-2:]),                              # final quad split by 5000 blanks
        cat(textp[:-1], sp(4096), textp[-1:], np.frombuffer(b"\r\n\r\n", np.uint8)),  # trailing CRLFs
        cat(text[:4095], sp(1), text[4095:]),                               # a quad split at the chunk edge
        cat(sp(4093), text),                                                # G % 4 != 0 everywhere
    ]
    bad = []
    for t in cases[:3]:
        t = t.copy()
        keep = np.nonzero(t != ord(" "))[0]
        t[keep[4097 if keep.size > 4097 else 1]] = ord("*")  # a char read by the look-ahead
        bad.append(t)
        t2 = t.copy()
        t2[keep[keep.size // 2]] = ord("=")                  # '=' in the middle
        bad.append(t2)
    t = cases[2].copy()
    t[np.nonzero(t != ord(" "))[0][-3]] = ord("A")          # final quad 'xA==' non-canonical
    bad.append(t)
    t = cases[2].copy()
    t[np.nonzero(t != ord(" "))[0][-2]] = ord("A")          # 'xxA=': not canonical or bad bits
    bad.append(t)
    t = cases[2].copy()
    t[np.nonzero(t != ord(" "))[0][-1]] = ord("A")          # 'xx=A': data after padding
    bad.append(t)
    # near misses of the whitespace set (the kernels' arithmetic test must not skip them): each
    # is an invalid char at its position; and every whitespace byte at every lane offset
    for k, nb in enumerate((0x08, 0x0E, 0x1F, 0x21, 0x89, 0x8A, 0x8D, 0xA0, 0x00, 0x7F, 0xC9)):
        t = cat(text[:3000], np.frombuffer(b"\r\n", np.uint8), text[3000:]).copy()
        t[1000 + 37 * k] = nb
        bad.append(t)
    allws = np.frombuffer(b" \t\n\r\x0b\x0c", np.uint8)
    t = np.concatenate([cat(text[i: i + 5], allws[i % 6: i % 6 + 1 + (i % 3)]) for i in range(0, 8000, 5)])
    bad.append(cat(t, text[8000:]))
    for i, t in enumerate(cases + bad):
        ref, rerr, rst = oracle.decode_ws(t)
        for off in (0, 1):
            out, err = b64.decode_ws(to_dev(t, off))
            assert err == rerr, (i, off, err, rerr, rst)
            assert np.array_equal(out.cpu().numpy(), ref), (i, off)
        refl, rerrl, _ = oracle.decode_ws(t, lenient=True)
        out, err = b64.decode_ws(to_dev(t), b64.lenient_of(b64.standard()))
        assert err == rerrl and np.array_equal(out.cpu().numpy(), refl), i


# ------------------------------------------------------------------ streaming (carry between calls)

def _splits(total: int, rng, small: bool):
    """Piece lengths summing to total: tiny pieces (0-9) when small, else a mix of tiny,
    chunk-sized and odd multi-chunk pieces."""
    out, left = [], total
    while left > 0:
        if small or rng.random() < 0.4:
            k = int(rng.integers(0, 10))
        else:
            k = int(rng.choice([1024, 4096, 3 * 1024 + 1, 100_003, 768 * 50 + 7, 1 << 16]))
        k = min(k, left)
        out.append(k)
        left -= k
        if rng.random() < 0.05:
            out.append(0)
    return out


def test_encode_stream_vs_oracle(b64):
    """Streaming encode (R15): any split of the input gives the one-shot encode."""
    al = _alphabets(b64)
    rng = np.random.default_rng(21)
    for trial, n in enumerate([0, 1, 2, 3, 4, 5, 47, 1000, 100_000, 768 * 300 + 2, 1 << 20]):
        for small in ((True, False) if n < 5000 else (False,)):
            chars, pad, alpha = al[trial % len(al)]
            x = synth.data(n, seed=300 + trial)
            dx = to_dev(x)
            es = b64.EncodeStream(alpha)
            parts, pos = [], 0
            for k in _splits(n, rng, small):
                parts.append(es.update(dx[pos: pos + k]).cpu().numpy())
                pos += k
            parts.append(es.end().cpu().numpy())
            got = np.concatenate(parts)
            assert np.array_equal(got, oracle.encode(x, chars, pad)), (n, small)
            assert es.st.produced == got.size == b64.encoded_len(n)


def _dec_stream(b64, text, alpha, pieces, misalign=0):
    ds = b64.DecodeStream(alpha)
    dt = to_dev(text, misalign)
    parts, pos = [], 0
    for k in pieces:
        parts.append(ds.update(dt[pos: pos + k]).cpu().numpy())
        pos += k
    tail, info = ds.end()
    parts.append(tail.cpu().numpy())
    return np.concatenate(parts), info.tolist()


def test_decode_stream_vs_oracle(b64):
    """Streaming decode: any split gives the one-shot decode -- output, err_off, status and
    out_len of the whole text -- including errors in straddling quads, in the held-back
    final quad and the LENGTH rule."""
    al = _alphabets(b64)
    rng = np.random.default_rng(22)
    cases = 0
    for trial, n in enumerate([0, 1, 2, 3, 4, 30, 31, 32, 1000, 100_000, 768 * 300 + 1, 1 << 20]):
        chars, pad, alpha = al[trial % len(al)]
        text = oracle.encode(synth.data(n, seed=400 + trial), chars, pad)
        variants = [text]
        if text.size > 8:
            for j in range(3):  # corrupted copies
                t2 = text.copy()
                p_, b_ = synth.corruption(1 + j, text.size, chars, seed=trial * 10 + j, pad=pad)
                t2[p_] = b_
                variants.append(t2)
            t3 = text.copy()  # a pad in the middle; bad final quad forms
            t3[text.size // 2] = pad
            variants.append(t3)
            t4 = text.copy()
            t4[-1] = ord("*")
            variants.append(t4)
            variants.append(text[:-1])  # LENGTH (m % 4 == 3)
            variants.append(text[:-3])  # LENGTH (m % 4 == 1)
        for v in variants:
            ref, rerr, rst = oracle.decode(v, chars, pad)
            for small in ((True, False) if v.size < 5000 else (False,)):
                got, (err, st, olen) = _dec_stream(b64, v, alpha, _splits(v.size, rng, small), misalign=trial % 3)
                assert (err, st) == (rerr, rst), (n, small, err, st, rerr, rst)
                assert olen == ref.size, (n, olen, ref.size)
                assert np.array_equal(got[:olen], ref), n
                cases += 1
    assert cases > 60


def test_decode_stream_error_at_every_boundary_position(b64):
    """Piece boundary at every offset of a small text x one bad char at every position:
    the error lands in the join quad, a bulk quad or the held final quad."""
    text = oracle.encode(synth.data(45, seed=9))  # 60 chars, final quad 'xxxx'
    std = b64.standard()
    for cut in range(0, text.size + 1, 3):
        for p in range(0, text.size, 5):
            t = text.copy()
            t[p] = ord("$")
            _, rerr, rst = oracle.decode(t)
            got, (err, st, olen) = _dec_stream(b64, t, std, [cut, text.size - cut])
            assert (err, st) == (rerr, rst) == (p, oracle.ST_BADCHAR), (cut, p)


# ------------------------------------------------------------------ lenient decode (R16)

def _noncanonical_texts(chars, pad, n_list=(1, 2, 4, 5, 700, 3000, 200_000, 600_001)):
    """Valid texts whose final quad is 'xx==' / 'xxx=' with NON-zero trailing bits (strict
    rejects them as NONCANON at m-3 / m-2; lenient drops the bits), plus their canonical form."""
    out = []
    for n in n_list:
        t = oracle.encode(synth.data(n, seed=n), chars, pad)
        out.append(t)
        if n % 3:
            u = t.copy()
            k = t.size - (3 if n % 3 == 1 else 2)       # the char before the padding
            v = chars.index(bytes([u[k]]))
            u[k] = chars[v | (1 if n % 3 == 2 else 5)]  # set dropped low bits
            out.append(u)
    return out


def test_lenient_decode_all_paths_vs_oracle(b64):
    """B64_ALPHA_LENIENT honoured by every decode entry point: single call (small cluster and
    bulk paths), misaligned generic, chunk API, group, batch, stream, unpadded, whitespace."""
    al = _alphabets(b64)
    for ai in (0, 1, 3):
        chars, pad, strict_a = al[ai]
        len_a = b64.lenient_of(strict_a)
        texts = _noncanonical_texts(chars, pad)
        for t in texts:
            ref, rerr, rst = oracle.decode(t, chars, pad, lenient=True)
            sref = oracle.decode(t, chars, pad)
            for oi, oo in ((0, 0), (1, 3)):
                assert dec_check_lenient(b64, t, ref, rerr, rst, len_a, oi, oo)
            # strict alphabet still strict
            out, info = b64.decode_async(to_dev(t), strict_a)
            assert tuple(info.tolist()[:2]) == (sref[1], sref[2])
            # chunk API as 3 shards (+ finalize)
            if t.size >= 12:
                cut = (t.size // 3) // 4 * 4
                dt = to_dev(t)
                cell = torch.full((1,), b64.ERR_NONE, dtype=torch.int64, device=DEV)
                o = torch.empty(3 * (t.size // 4) + 3, dtype=torch.uint8, device=DEV)
                b64.decode_chunk(dt[:cut], 0, False, cell, len_a, out=o[: 3 * cut // 4])
                b64.decode_chunk(dt[cut:], cut, True, cell, len_a, out=o[3 * cut // 4:])
                eo = torch.empty(1, dtype=torch.int64, device=DEV)
                b64.decode_finalize(cell, eo)
                assert int(eo.item()) == rerr
                if rerr < 0:
                    assert np.array_equal(o[: ref.size].cpu().numpy(), ref)
            # streaming
            got, (err, st, olen) = _dec_stream(b64, t, len_a, [t.size // 2, t.size - t.size // 2])
            assert (err, st, olen) == (rerr, rst, ref.size) and np.array_equal(got[:olen], ref)
            # unpadded (the same text with its '=' removed)
            bare = t[: t.size - int((t[-2:] == pad).sum())] if t.size else t
            uref = oracle.decode_unpadded(bare, chars, pad, lenient=True)
            if bare.size % 4 != 1:
                uo, uerr = b64.decode_unpadded(to_dev(bare), len_a)
                assert uerr == uref[1] and np.array_equal(uo.cpu().numpy(), uref[0])
            # whitespace-skipping
            if t.size:
                wt = np.concatenate([t[:1], np.frombuffer(b"\r\n", np.uint8), t[1:]])
                wref = oracle.decode_ws(wt, chars, pad, lenient=True)
                wo, werr = b64.decode_ws(to_dev(wt), len_a)
                assert werr == wref[1] and np.array_equal(wo.cpu().numpy(), wref[0])
        # group and batch over all texts at once
        douts, err, st = b64.decode_group([to_dev(t) for t in texts], len_a)
        errc, stc = err.cpu().numpy(), st.cpu().numpy()
        lens = np.array([t.size for t in texts], dtype=np.int64)
        in_off = np.zeros(len(texts) + 1, dtype=np.int64)
        np.cumsum(lens, out=in_off[1:])
        cat = np.concatenate(texts)
        bo, boff, bst, berr, bolen = b64.decode_batch(to_dev(cat), torch.from_numpy(in_off).to(DEV), len_a)
        bst, berr, bolen, boff = bst.cpu().numpy(), berr.cpu().numpy(), bolen.cpu().numpy(), boff.cpu().numpy()
        bo = bo.cpu().numpy()
        for i, t in enumerate(texts):
            ref, rerr, rst = oracle.decode(t, chars, pad, lenient=True)
            assert (errc[i], stc[i]) == (rerr, rst), i
            assert np.array_equal(douts[i][: ref.size].cpu().numpy(), ref), i
            assert (berr[i], bst[i], bolen[i]) == (rerr, rst, ref.size), i
            assert np.array_equal(bo[boff[i]: boff[i] + ref.size], ref), i


def dec_check_lenient(b64, text, ref, rerr, rst, alpha, off_in, off_out):
    t = to_dev(text, off_in)
    cap = 3 * (text.size // 4)
    obuf = torch.empty(cap + off_out + 64, dtype=torch.uint8, device=DEV)
    out, info = b64.decode_async(t, alpha, out=obuf[off_out: off_out + max(cap, 1)])
    err, st, olen = info.tolist()
    assert (err, st, olen) == (rerr, rst, ref.size), (text.size, err, st, rerr, rst)
    assert np.array_equal(out[:olen].cpu().numpy(), ref)
    return True


def test_lenient_every_byte_final_quad(b64):
    """Every byte value at each final-quad position of 'xxxx' / 'xx==' / 'xxx=' texts with a
    lenient alphabet (the single-launch small path) vs the lenient oracle."""
    len_a = b64.lenient_of(b64.standard())
    for raw_len in (30, 31, 32):
        text = oracle.encode(synth.data(raw_len, seed=raw_len))
        for p in range(text.size - 4, text.size):
            for v in range(256):
                t = text.copy()
                t[p] = v
                ref, rerr, rst = oracle.decode(t, lenient=True)
                dec_check_lenient(b64, t, ref, rerr, rst, len_a, 0, 0)


# ------------------------------------------------------------------ one-sided peer combine (f4)

def _packed_words(rng, n, none_frac=0.3):
    pos = rng.integers(0, 1 << 40, n, dtype=np.int64)
    kind = rng.integers(1, 4, n, dtype=np.int64)
    w = (pos << 3) | kind
    w[rng.random(n) < none_frac] = b64_err_none()
    return w


def b64_err_none():
    return 0x7F7F7F7F7F7F7F7F


def _api_form(words):
    w = np.asarray(words, dtype=np.int64)
    none = w >= b64_err_none()
    return np.where(none, -1, w >> 3), np.where(none, 0, w & 7).astype(np.int32)


def test_peer_combine_emulated_ranks(b64):
    """W ranks emulated on one GPU (one cooperative kernel, block r = rank r) through E
    back-to-back epochs: every rank sees the MIN over ranks of that epoch's words (the slot
    parity and epoch tags of b64_peer_combine's push protocol, real system-scope stores)."""
    L = b64._lib.lib()
    rng = np.random.default_rng(5)
    for world, K, epochs in ((1, 6, 5), (2, 6, 9), (3, 1, 7), (8, 6, 12), (5, 40, 4)):
        nbytes = int(L.b64_peer_combine_bytes(K))
        bufs = [torch.empty(nbytes, dtype=torch.uint8, device=DEV) for _ in range(world)]
        for bb in bufs:
            b64._lib.check(L.b64_peer_combine_init(ctypes.c_void_p(bb.data_ptr()), K, None), "init")
        d_bufs = torch.tensor([bb.data_ptr() for bb in bufs], dtype=torch.int64, device=DEV)
        local = _packed_words(rng, epochs * world * K).reshape(epochs, world, K)
        local[0, :, 0] = b64_err_none()  # an epoch-0 stream with no error anywhere
        d_local = torch.from_numpy(local.copy()).to(DEV)
        d_out = torch.zeros(epochs * world * K, dtype=torch.int64, device=DEV)
        ok = torch.ones(1, dtype=torch.int32, device=DEV)
        b64._lib.check(L.b64_peer_combine_emulate(ctypes.c_void_p(d_bufs.data_ptr()), world,
                                                  ctypes.c_void_p(d_local.data_ptr()), K, epochs,
                                                  ctypes.c_void_p(d_out.data_ptr()),
                                                  ctypes.c_void_p(ok.data_ptr()), None), "emulate")
        torch.cuda.synchronize()
        assert int(ok.item()) == 1
        got = d_out.cpu().numpy().reshape(epochs, world, K)
        want = local.min(axis=1)
        for r in range(world):
            assert np.array_equal(got[:, r, :], want), (world, K, r)
        # after the epochs, slot e & 1 of every rank's buffer holds epoch e's words of every rank
        # as cells {low / high 32-bit half, tag e + 1} (e = the last two epochs)
        for bb in bufs:
            raw = bb.cpu().numpy().view(np.uint64).reshape(2, 32, K, 2)
            for e in range(max(0, epochs - 2), epochs):
                cells = raw[e & 1, :world]
                assert np.all(cells >> np.uint64(32) == np.uint64(e + 1)), (world, K, e)
                words = (cells[..., 1] << np.uint64(32)) | (cells[..., 0] & np.uint64(0xFFFFFFFF))
                assert np.array_equal(words.view(np.int64), local[e]), (world, K, e)


def test_codec_fused_peer_world1(b64):
    """b64_codec_group_fused_peer at world 1 (dist.PeerCombine.codec_fused): the codec kernel's
    last CTA runs the peer-memory MIN protocol before it finalises; results equal the oracle,
    epoch after epoch, and the error words / ticket are left ready."""
    from paper_1910_05109_b200 import dist as b64dist

    xs = [synth.data(n, seed=80 + n) for n in (1 << 20, 768 * 7 + 2, 3)]
    refs = [oracle.encode(x) for x in xs]
    dx = [to_dev(x) for x in xs]
    pc = b64dist.PeerCombine(len(xs))
    try:
        cells = torch.full((len(xs),), b64.ERR_NONE, dtype=torch.int64, device=DEV)
        ticket = torch.zeros(1, dtype=torch.int32, device=DEV)
        for e in range(5):
            texts = [r.copy() for r in refs]
            if e % 2:
                texts[0][1000 + e] = ord("!")
                texts[2][-1] = ord("?")
            dt = [to_dev(t) for t in texts]
            eitems, eouts = b64._enc_items(dx, None, None)
            ditems, douts, _ = b64._dec_items(dt, None, None, cells, None, None)
            err = torch.empty(len(xs), dtype=torch.int64, device=DEV)
            st = torch.empty(len(xs), dtype=torch.int32, device=DEV)
            pc.codec_fused(eitems, len(xs), ditems, err, st, ticket)
            torch.cuda.synchronize()
            for i in range(len(xs)):
                assert np.array_equal(eouts[i].cpu().numpy(), refs[i]), (e, i)
                ref, rerr, rst = oracle.decode(texts[i])
                assert (int(err[i].item()), int(st[i].item())) == (rerr, rst), (e, i)
                assert np.array_equal(douts[i][: ref.size].cpu().numpy(), ref), (e, i)
            assert torch.all(cells == b64.ERR_NONE) and int(ticket.item()) == 0
    finally:
        pc.close()


def test_peer_combine_world1_api(b64):
    """dist.PeerCombine at world 1 (the per-rank kernel, IPC-allocated buffer): err_off/status
    equal b64_decode_finalize_n of the same words, epoch after epoch."""
    from paper_1910_05109_b200 import dist as b64dist

    rng = np.random.default_rng(6)
    pc = b64dist.PeerCombine(6)
    try:
        for e in range(6):
            w = _packed_words(rng, 6)
            cells = torch.from_numpy(w).to(DEV)
            err = torch.empty(6, dtype=torch.int64, device=DEV)
            st = torch.empty(6, dtype=torch.int32, device=DEV)
            pc.combine(cells, err, st)
            torch.cuda.synchronize()
            we, ws = _api_form(w)
            assert np.array_equal(err.cpu().numpy(), we), e
            assert np.array_equal(st.cpu().numpy(), ws), e
        assert pc.validate()  # the bench's collective self-test (world 1: the own buffer only)
    finally:
        pc.close()
