"""compute-sanitizer subset: every C-ABI entry point at
small sizes -- fast and generic kernels, the single-launch cluster kernels, the fused
last-CTA finalize, the stream joins, the whitespace paths, the batch kernels and offsets, the
emulated peer combine -- each result checked against the oracle.

Meant for the four compute-sanitizer tools (tools/sanitize.sh).  compute-sanitizer was closed on
this project's GPU pool (runs under it left GPUs needing a reset), so the bounds check is done
by the hardware instead (tests/test_guard_pages.py: every buffer against an unmapped page);
this file still runs in the plain `-m gpu` pass.  With the tool:

    PYTORCH_NO_CUDA_MEMORY_CACHING=1 compute-sanitizer --tool memcheck \\
        python -m pytest tests/test_sanitize.py -m sanitize -q

With the caching allocator off every tensor is its own cudaMalloc, so memcheck sees the
exact allocation bounds of every input and output.  Marked gpu as well: the plain `-m gpu`
run executes it too (quickly, without the tool)."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.sanitize]

DEV = "cuda:0"


@pytest.fixture(scope="module")
def b64():
    import __graft_entry__ as g

    g.build()
    import paper_1910_05109_b200 as m

    return m


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _exact(n, off=0):
    """A device tensor that is exactly its own allocation (n bytes) when caching is off, at an
    offset inside a slightly larger allocation otherwise (off > 0: misaligned start)."""
    if off == 0:
        return torch.empty(max(n, 1), dtype=torch.uint8, device=DEV)[:n]
    return torch.empty(n + off, dtype=torch.uint8, device=DEV)[off:]


SIZES = (0, 1, 2, 3, 4, 5, 47, 48, 49, 767, 768, 769, 3000, 70_001)


def test_encode_decode_single(b64):
    for n in SIZES:
        x = synth.data(n, seed=n)
        ref = oracle.encode(x)
        for off in (0, 1):
            xd = _exact(n, off)
            xd.copy_(_t(x)) if n else None
            od = _exact(ref.size, 3 * off)
            b64.encode(xd, out=od)
            assert np.array_equal(od.cpu().numpy(), ref), (n, off)
            td = _exact(ref.size, 5 * off)
            td.copy_(_t(ref)) if ref.size else None
            y, err = b64.decode(td)
            assert err == -1 and np.array_equal(y.cpu().numpy(), x), (n, off)
            if ref.size >= 8:
                t2 = ref.copy()
                t2[ref.size // 2] = ord("*")
                td.copy_(_t(t2))
                _, err = b64.decode(td)
                assert err == oracle.decode(t2)[1]


def test_decode_variants(b64):
    x = synth.data(900_001, seed=1)  # above the single-launch cluster size: fast kernel + fused ctx
    ref = oracle.encode(x)
    td = _t(ref)
    y, err = b64.decode(td, ctx=b64.DecodeContext())
    assert err == -1 and np.array_equal(y.cpu().numpy(), x)
    out, info = b64.decode_async(td)
    assert info.tolist()[0] == -1
    for n in (2, 3, 5, 1000):
        xs = synth.data(n, seed=n)
        tu = oracle.encode_unpadded(xs, oracle.URL)
        y, err = b64.decode_unpadded(_t(tu), b64.url())
        assert err == -1 and np.array_equal(y.cpu().numpy(), xs)
    lenient = b64.lenient_of(b64.standard())
    y, err = b64.decode(_t(oracle.encode(x[:1000])), lenient)
    assert err == -1
    cell = torch.full((1,), b64.ERR_NONE, dtype=torch.int64, device=DEV)
    b64.decode_chunk(td[:4096], 0, False, cell)
    eo = torch.empty(1, dtype=torch.int64, device=DEV)
    b64.decode_finalize(cell, eo)
    assert int(eo.item()) == -1


def test_decode_ws_paths(b64):
    x = synth.data(600_000, seed=2)
    t = oracle.encode(x)
    mime = np.concatenate([np.concatenate([t[i: i + 76], np.frombuffer(b"\r\n", np.uint8)])
                           for i in range(0, t.size, 76)])
    for text in (mime[:5000], mime, np.concatenate([mime[:1000], [32], mime[1000:]]).astype(np.uint8)):
        y, err = b64.decode_ws(_t(text))
        ref, rerr, _ = oracle.decode_ws(text)
        assert err == rerr and np.array_equal(y.cpu().numpy(), ref)


def test_streams(b64):
    x = synth.data(200_003, seed=3)
    ref = oracle.encode(x)
    es = b64.EncodeStream()
    cuts = (0, 1, 2, 5, 100_000, 200_003)
    parts = [es.update(_t(x[a:b])) for a, b in zip(cuts, cuts[1:])] + [es.end()]
    assert np.array_equal(torch.cat(parts).cpu().numpy(), ref)
    ds = b64.DecodeStream()
    cuts = (0, 1, 3, 7, 150_001, ref.size)
    parts = [ds.update(_t(ref[a:b])) for a, b in zip(cuts, cuts[1:])]
    tail, info = ds.end()
    torch.cuda.synchronize()
    got = torch.cat(parts + [tail]).cpu().numpy()
    assert info.tolist()[0] == -1 and np.array_equal(got[: x.size], x)


def test_groups(b64):
    xs = [synth.data(n, seed=n) for n in (300_001, 4096, 768 * 5)]
    refs = [oracle.encode(v) for v in xs]
    texts = [r.copy() for r in refs]
    texts[1][100] = ord("*")
    dx = [_t(v) for v in xs]
    dt = [_t(v) for v in texts]
    eo = b64.encode_group(dx)
    assert all(np.array_equal(a.cpu().numpy(), r) for a, r in zip(eo, refs))
    do, err, st = b64.decode_group(dt)
    assert err.tolist() == [-1, 100, -1]
    eo, do, err, st = b64.codec_group(dx, dt)
    assert err.tolist() == [-1, 100, -1]
    eo, do, err, st = b64.codec_group_fused(dx, dt)
    assert err.tolist() == [-1, 100, -1]
    assert all(np.array_equal(a.cpu().numpy(), r) for a, r in zip(eo, refs))


def test_batches(b64):
    Ls = synth.loguniform_lengths(3000, hi=4096, seed=4)
    off = synth.offsets(Ls)
    x = synth.data(int(off[-1]), seed=4)
    ref, roff = oracle.encode_batch(x, off)
    out, oo = b64.encode_batch(_t(x), _t(off))
    assert np.array_equal(oo.cpu().numpy(), roff) and np.array_equal(out[: ref.size].cpu().numpy(), ref)
    t = ref.copy()
    t[roff[7] + 1] = ord("*")
    rout, rdoff, rst, rerr, rlen = oracle.decode_batch(t, roff)
    o, doo, st, err, olen = b64.decode_batch(_t(t), _t(roff))
    assert np.array_equal(st.cpu().numpy(), rst) and np.array_equal(err.cpu().numpy(), rerr)
    assert np.array_equal(olen.cpu().numpy(), rlen)


def test_host_pipeline(b64):
    pipe = b64.HostPipeline(chunk_bytes=3072 * 2)
    x = synth.data(20_000, seed=5)
    t = pipe.encode(torch.from_numpy(x).pin_memory())
    assert np.array_equal(t.numpy(), oracle.encode(x))
    y, err = pipe.decode(t.clone().pin_memory())
    assert err == -1 and np.array_equal(y.numpy(), x)


def test_peer_combine_emulated(b64):
    from paper_1910_05109_b200 import _lib

    L = _lib.lib()
    world, count, epochs = 4, 3, 2
    nb = int(L.b64_peer_combine_bytes(count))
    bufs = [torch.empty(nb, dtype=torch.uint8, device=DEV) for _ in range(world)]
    for b in bufs:
        _lib.check(L.b64_peer_combine_init(ctypes.c_void_p(b.data_ptr()), count, None), "init")
    ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=DEV)
    rng = np.random.default_rng(0)
    local = rng.integers(0, 1 << 40, size=(epochs, world, count)).astype(np.int64)
    dl = _t(local.reshape(-1))
    out = torch.empty(epochs * world * count, dtype=torch.int64, device=DEV)
    ok = torch.ones(1, dtype=torch.int32, device=DEV)
    _lib.check(L.b64_peer_combine_emulate(ctypes.c_void_p(ptrs.data_ptr()), world, ctypes.c_void_p(dl.data_ptr()),
                                          count, epochs, ctypes.c_void_p(out.data_ptr()),
                                          ctypes.c_void_p(ok.data_ptr()), None), "emulate")
    torch.cuda.synchronize()
    assert int(ok.item()) == 1
    got = out.cpu().numpy().reshape(epochs, world, count)
    for e in range(epochs):
        for r in range(world):
            assert np.array_equal(got[e, r], local[e].min(axis=0))
