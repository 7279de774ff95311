"""Back-to-back dependent operations on ONE stream with no host synchronisation in between:
each op reads what the kernel launched just before it wrote, so a load scheduled before
griddepcontrol.wait (the programmatic-dependent-launch hazard tests/test_pdl_order.py checks
statically) would read stale bytes here.  Buffers are reused across rounds and pre-filled with
garbage on the device right before each producer, so stale data cannot pass by accident."""
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

    return m


def test_dependent_chain_no_sync(b64):
    rng = np.random.default_rng(123)
    cap = 3 << 20
    xbuf = torch.empty(cap + 64, dtype=torch.uint8, device=DEV)
    tbuf = torch.empty(4 * cap // 3 + 128, dtype=torch.uint8, device=DEV)
    ybuf = torch.empty(cap + 64, dtype=torch.uint8, device=DEV)
    t2buf = torch.empty(4 * cap // 3 + 128, dtype=torch.uint8, device=DEV)
    sbuf = torch.empty(cap + 64, dtype=torch.uint8, device=DEV)
    ctx = b64.DecodeContext()
    for rnd in range(12):
        n = int(rng.integers(1, cap)) if rnd % 3 else int(rng.integers(1, 5000))
        xo, to, yo, t2o = (int(v) for v in rng.integers(0, 32, 4))
        x = synth.data(n, seed=500 + rnd)
        m = int(b64.encoded_len(n))
        xd = xbuf[xo: xo + n]
        xd.copy_(torch.from_numpy(x))
        # garbage everywhere first (torch fills are kernels too: none may sit between a producer
        # and its consumer below), and the objects whose set-up launches work
        for b in (tbuf, ybuf, t2buf, sbuf):
            b.fill_(0xEE)
        info = b64.new_info()
        ds = b64.DecodeStream()
        piece = int(rng.integers(7, 400_000))
        # 1. encode
        t = b64.encode(xd, out=tbuf[4 * (to // 4): 4 * (to // 4) + m])
        # 2. decode what 1 wrote (fused single launch with a context, no sync)
        y, info = b64.decode_async(t, out=ybuf[16 * (yo // 16): 16 * (yo // 16) + b64.decoded_len_max(m)],
                                   info=info, ctx=ctx)
        # 3. encode what 2 wrote, at a misaligned output (the unaligned fast kernel above 64 Ki)
        t2 = b64.encode(y[:n], out=t2buf[4 * (t2o // 4) + 4: 4 * (t2o // 4) + 4 + m])
        # 4. stream-decode what 3 wrote, in odd pieces, into one buffer
        o = p = 0
        while p < m:
            k = min(piece, m - p)
            c = ds.out_len(k)
            ds.update(t2[p: p + k], out=sbuf[o: o + max(c, 1)])
            o += c
            p += k
        _, sinfo = ds.end(out=sbuf[o: o + max(ds.end_len(), 1)])
        # 5. grouped encode of what 4 wrote and of x, in one launch
        e1, e2 = b64.encode_group([sbuf[:n], xd])
        torch.cuda.synchronize()
        ref_t = oracle.encode(x)
        assert np.array_equal(t.cpu().numpy(), ref_t), (rnd, "encode")
        err, _, olen = info.tolist()
        assert err == -1 and olen == n and np.array_equal(y[:n].cpu().numpy(), x), (rnd, "decode")
        assert np.array_equal(t2.cpu().numpy(), ref_t), (rnd, "re-encode")
        serr, _, solen = sinfo.tolist()
        assert serr == -1 and solen == n and np.array_equal(sbuf[:n].cpu().numpy(), x), (rnd, "stream")
        assert np.array_equal(e1.cpu().numpy(), ref_t) and np.array_equal(e2.cpu().numpy(), ref_t), (rnd, "group")
