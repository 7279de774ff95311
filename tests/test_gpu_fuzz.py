"""Property-based GPU fuzzing (hypothesis): random lengths, alignments, alphabets (incl.
lenient), corruptions and entry points -- every result compared with the oracle, element
by element.  Seeded (derandomized) so a failure reproduces."""

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
import synth

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
SETTINGS = settings(max_examples=400, deadline=None, derandomize=True,
                    suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])


@pytest.fixture(scope="module")
def b64():
    import __graft_entry__ as g

    g.build()
    import paper_1910_05109_b200 as m

    return m


def _alpha(b64, kind, seed):
    if kind == "std":
        return oracle.STANDARD, oracle.PAD, b64.standard()
    if kind == "url":
        return oracle.URL, oracle.PAD, b64.url()
    rng = np.random.default_rng(seed)
    perm = rng.permutation(127)[:65]
    chars, pad = bytes(perm[:64].tolist()), int(perm[64])
    return chars, pad, b64.alphabet(chars, bytes([pad]))


def _dev(x, off):
    buf = torch.empty(x.size + off + 64, dtype=torch.uint8, device=DEV)
    t = buf[off: off + x.size]
    if x.size:
        t.copy_(torch.from_numpy(x))
    return t


lengths = st.one_of(st.integers(0, 40), st.integers(0, 5000), st.integers(760, 800), st.integers(0, 300_000))


@SETTINGS
@given(n=lengths, kind=st.sampled_from(["std", "url", "custom"]), aseed=st.integers(0, 50),
       off_in=st.sampled_from([0, 0, 1, 3, 8]), off_out=st.sampled_from([0, 0, 1, 2, 16]),
       lenient=st.booleans(), k_bad=st.integers(0, 3), seed=st.integers(0, 10_000),
       api=st.sampled_from(["single", "ctx", "chunk", "group", "codec", "stream", "batch", "unpadded", "ws",
                            "ws_lines", "consume", "stream_overlap"]))
def test_fuzz_encode_decode_vs_oracle(b64, n, kind, aseed, off_in, off_out, lenient, k_bad, seed, api):
    chars, pad, alpha = _alpha(b64, kind, aseed)
    if lenient:
        alpha = b64.lenient_of(alpha)
    x = synth.data(n, seed=seed)
    ref_t = oracle.encode(x, chars, pad)
    text = ref_t.copy()
    if k_bad and text.size:
        pos, bad = synth.corruption(min(k_bad, text.size), text.size, chars, seed=seed, pad=pad)
        text[pos] = bad
        if seed % 5 == 0 and text.size >= 4:
            text[-4 + seed % 4] = pad  # a misplaced pad in the final quad
    ref, rerr, rst = oracle.decode(text, chars, pad, lenient=lenient)
    m = text.size
    if api == "ctx":  # one-launch decode with a self-resetting context (b64_decode_fused)
        if not hasattr(b64, "_fuzz_ctx"):
            b64._fuzz_ctx = b64.DecodeContext()
        # a valid unpadded prefix (n % 3 == 0) takes the text past the single-cluster size, so
        # the fused kernel runs; the expected result is the oracle's on the concatenation
        pre = oracle.encode(synth.data(3 * (200_000 + seed), seed=seed + 1), chars, pad)
        text = np.concatenate([pre, text])
        ref, rerr, rst = oracle.decode(text, chars, pad, lenient=lenient)
        m = text.size
        obuf = torch.empty(3 * (m // 4) + off_out + 8, dtype=torch.uint8, device=DEV)
        out, info = b64.decode_async(_dev(text, off_in), alpha, out=obuf[off_out: off_out + max(3 * (m // 4), 1)],
                                     ctx=b64._fuzz_ctx)
        err, stt, olen = info.tolist()
        got = out[:olen].cpu().numpy()
    elif api == "single":
        t = b64.encode(_dev(x, off_in), alpha, out=torch.empty(m + off_out + 8, dtype=torch.uint8,
                                                               device=DEV)[off_out:])
        assert np.array_equal(t.cpu().numpy(), ref_t)
        obuf = torch.empty(3 * (m // 4) + off_out + 8, dtype=torch.uint8, device=DEV)
        out, info = b64.decode_async(_dev(text, off_in), alpha, out=obuf[off_out: off_out + max(3 * (m // 4), 1)])
        err, stt, olen = info.tolist()
        got = out[:olen].cpu().numpy()
    elif api == "chunk":
        cut = (m // 3) // 4 * 4
        dt = _dev(text, off_in)
        cell = torch.full((1,), b64.ERR_NONE, dtype=torch.int64, device=DEV)
        o = torch.empty(3 * (m // 4) + 8, dtype=torch.uint8, device=DEV)
        if m:
            b64.decode_chunk(dt[:cut], 0, False, cell, alpha, out=o[: 3 * cut // 4 + 1])
            b64.decode_chunk(dt[cut:], cut, True, cell, alpha, out=o[3 * cut // 4:])
        eo = torch.empty(1, dtype=torch.int64, device=DEV)
        sto = torch.zeros(1, dtype=torch.int32, device=DEV)
        b64.decode_finalize(cell, eo, sto)
        err, stt = int(eo.item()), int(sto.item())
        olen = ref.size if err < 0 else 3 * (err // 4)
        got = o[:olen].cpu().numpy()
    elif api in ("group", "codec"):
        dx, dt = _dev(x, off_in), _dev(text, off_in)
        if api == "group":
            (eo,) = b64.encode_group([dx], alpha)
            (o,), e, s = b64.decode_group([dt], alpha)
        else:
            (eo,), (o,), e, s = b64.codec_group([dx], [dt], alpha, alpha)
        assert np.array_equal(eo.cpu().numpy(), ref_t)
        err, stt = int(e.item()), int(s.item())
        olen = ref.size if err < 0 else 3 * (err // 4)
        got = o[:olen].cpu().numpy()
    elif api == "stream":
        es, ds = b64.EncodeStream(alpha), b64.DecodeStream(alpha)
        dx, dt = _dev(x, off_in), _dev(text, off_in)
        rng = np.random.default_rng(seed)
        parts, p = [], 0
        while p < n:
            k = int(rng.integers(0, 5000))
            parts.append(es.update(dx[p: p + k]).cpu().numpy())
            p += k
        parts.append(es.end().cpu().numpy())
        assert np.array_equal(np.concatenate(parts), ref_t)
        parts, p = [], 0
        while p < m:
            k = int(rng.integers(0, 7000))
            parts.append(ds.update(dt[p: p + k]).cpu().numpy())
            p += k
        tail, info = ds.end()
        parts.append(tail.cpu().numpy())
        err, stt, olen = info.tolist()
        got = np.concatenate(parts)[:olen]
    elif api == "stream_overlap":  # B64_STREAM_OVERLAP: large random pieces into one buffer, no sync between
        rng = np.random.default_rng(seed)
        pre = synth.data(3 * (100_000 + seed), seed=seed + 3)  # a prefix so that pieces reach the fast kernels
        x2 = np.concatenate([pre, x])
        ref_t2 = oracle.encode(x2, chars, pad)
        text = np.concatenate([oracle.encode(pre, chars, pad), text])
        ref, rerr, rst = oracle.decode(text, chars, pad, lenient=lenient)
        m = text.size
        es = b64.EncodeStream(alpha, overlap=True)
        dx = _dev(x2, off_in)
        eb = torch.full((ref_t2.size + 8,), 0xA5, dtype=torch.uint8, device=DEV)
        o = p = 0
        while p < x2.size:
            k = int(rng.integers(1, 200_000))
            c = es.out_len(k if p + k <= x2.size else x2.size - p)
            es.update(dx[p: p + k], out=eb[o: o + max(c, 1)])
            o += c
            p += k
        es.end(out=eb[o: o + max(es.end_len(), 1)])
        assert np.array_equal(eb[: ref_t2.size].cpu().numpy(), ref_t2), (api, n, seed)
        ds = b64.DecodeStream(alpha, overlap=True)
        dt = _dev(text, off_in)
        db = torch.full((3 * (m // 4) + 8,), 0xA5, dtype=torch.uint8, device=DEV)
        o = p = 0
        while p < m:
            k = min(int(rng.integers(1, 250_000)), m - p)
            c = ds.out_len(k)
            ds.update(dt[p: p + k], out=db[o: o + max(c, 1)])
            o += c
            p += k
        tail, info = ds.end(out=db[o: o + max(ds.end_len(), 1)])
        err, stt, olen = info.tolist()
        got = db[:olen].cpu().numpy()
    elif api == "unpadded":  # the same text with its '=' stripped (R13), one call
        t_u = text[: text.size - int(np.sum(text[-2:] == pad))] if text.size >= 4 else text
        if t_u.size % 4 == 1:
            return
        ref, rerr, rst = oracle.decode_unpadded(t_u, chars, pad, lenient=lenient)
        out, err = b64.decode_unpadded(_dev(t_u, off_in), alpha)
        assert err == rerr, (api, n, err, rerr, rst)
        assert np.array_equal(out.cpu().numpy(), ref)
        return
    elif api == "ws":  # the text with seeded whitespace runs inserted (R14)
        rng = np.random.default_rng(seed)
        k = int(rng.integers(0, 1 + text.size // 8))
        pos = np.sort(rng.integers(0, text.size + 1, k))
        ws = np.frombuffer(b" \t\n\r\x0b\x0c", np.uint8)
        t_w = np.insert(text, pos, ws[rng.integers(0, 6, k)]) if k else text
        if chars.translate(None, bytes(ws)) != chars:  # a whitespace char is data here: keep it simple
            return
        ref, rerr, rst = oracle.decode_ws(t_w, chars, pad, lenient=lenient)
        out, err = b64.decode_ws(_dev(t_w, off_in), alpha)
        assert err == rerr, (api, n, err, rerr, rst)
        assert np.array_equal(out.cpu().numpy(), ref)
        return
    elif api == "ws_lines":  # MIME-structured text above the one-launch size, with stray bytes (line segments)
        if chars.translate(None, b" \t\n\r\x0b\x0c") != chars:
            return
        rng = np.random.default_rng(seed)
        pre = oracle.encode(synth.data(3 * (150_000 + seed), seed=seed + 2), chars, pad)
        big = np.concatenate([pre, text])
        L = int(rng.choice([64, 76, 128]))
        sep = [b"\r\n", b"\n", b" "][seed % 3]
        lines = [big[i: i + L] for i in range(0, big.size, L)]
        t_l = np.concatenate([np.concatenate([ln, np.frombuffer(sep, np.uint8)]) for ln in lines])
        for _ in range(int(rng.integers(0, 5))):  # stray whitespace bytes / a doubled separator
            at = int(rng.integers(0, t_l.size))
            t_l = np.insert(t_l, at, np.frombuffer([b" ", b"\t", b"\n", b"\r\n"][int(rng.integers(0, 4))], np.uint8))
        ref, rerr, rst = oracle.decode_ws(t_l, chars, pad, lenient=lenient)
        out, err = b64.decode_ws(_dev(t_l, off_in), alpha)
        assert err == rerr, (api, n, err, rerr, rst, L, sep)
        assert np.array_equal(out.cpu().numpy(), ref), (api, n, L, sep)
        return
    elif api == "consume":  # decode -> consumer through a small ring, reassembled by the consumer
        full = torch.zeros(3 * (m // 4) + 8, dtype=torch.uint8, device=DEV)

        def consumer(chunk, off):
            full[off: off + chunk.numel()].copy_(chunk)

        ring = 3072 * (1 + seed % 7)
        err, olen = b64.decode_consume(_dev(text, off_in), consumer, alpha, ring_bytes=ring)
        assert err == rerr and (err >= 0 or olen == ref.size), (api, n, err, rerr)
        assert np.array_equal(full[: (olen if err < 0 else 3 * (err // 4))].cpu().numpy(),
                              ref[: (olen if err < 0 else 3 * (err // 4))])
        return
    else:  # batch of the text cut into pieces at random quad boundaries, plus the text itself
        rng = np.random.default_rng(seed)
        cuts = sorted(set([0, m] + [int(4 * v) for v in rng.integers(0, m // 4 + 1, 4)]))
        in_off = np.array(cuts + [m + m], dtype=np.int64)  # last string = the whole text again
        cat = np.concatenate([text, text])
        out, ooff, sts, errs, olens = b64.decode_batch(_dev(cat, off_in), torch.from_numpy(in_off).to(DEV), alpha)
        rout, rooff, rst_, rerr_, rolen = oracle.decode_batch(cat, in_off, chars, pad, lenient=lenient)
        assert np.array_equal(sts.cpu().numpy(), rst_) and np.array_equal(errs.cpu().numpy(), rerr_)
        assert np.array_equal(olens.cpu().numpy(), rolen)
        o = out.cpu().numpy()
        for i in range(len(rolen)):
            assert np.array_equal(o[rooff[i]: rooff[i] + rolen[i]], rout[rooff[i]: rooff[i] + rolen[i]]), i
        return
    assert (err, stt) == (rerr, rst), (api, n, err, stt, rerr, rst)
    assert olen == ref.size
    assert np.array_equal(got, ref)
