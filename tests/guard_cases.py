"""Guard-page bounds check of every C-ABI entry point (run by tests/test_guard_pages.py in a
subprocess: an out-of-bounds access faults the CUDA context, so the cases get a process of
their own).

compute-sanitizer is not available on this pool (runs under it left GPUs needing a reset),
so the bounds check is done with the hardware instead: every input, output, offsets array
and workspace of a case is placed in its own virtual-memory mapping (cuMemCreate /
cuMemMap) so that the buffer ENDS exactly at the end of the mapped range ("tail") or STARTS
exactly at its beginning ("head"), with the neighbouring virtual range reserved but unmapped.
Any read or write past the end (or before the start) of a buffer then touches an unmapped
page and raises an illegal-address fault instead of silently reading a neighbour's bytes.
The documented over-read of the generic kernels (b64gpu.h: whole 16-byte aligned blocks
that contain input bytes) never leaves the mapped page, so it is allowed by construction --
and any read of a block that holds NO input byte would fault here.

Every case also checks its results against the oracle.  Prints "ALL OK <n>" at the end.
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from cuda.bindings import driver as cu  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"driver call failed: {err}")
    return r[1] if isinstance(r, tuple) and len(r) == 2 else (r[1:] if isinstance(r, tuple) else None)


class Guarded:
    """n bytes of device memory ending ('tail') or starting ('head') at an unmapped page."""

    def __init__(self, n: int, where: str, dev: int = 0):
        prop = cu.CUmemAllocationProp()
        prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = dev
        gran = ck(cu.cuMemGetAllocationGranularity(
            prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM))
        self.gran = gran
        self.msz = max(gran, (max(n, 1) + gran - 1) // gran * gran)
        self.vsz = self.msz + 2 * gran
        self.va = int(ck(cu.cuMemAddressReserve(self.vsz, 0, 0, 0)))
        self.h = ck(cu.cuMemCreate(self.msz, prop, 0))
        ck(cu.cuMemMap(self.va + gran, self.msz, 0, self.h, 0))
        acc = cu.CUmemAccessDesc()
        acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = dev
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        ck(cu.cuMemSetAccess(self.va + gran, self.msz, [acc], 1))
        self.n = n
        self.ptr = self.va + gran + (self.msz - n if where == "tail" else 0)

    def put(self, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.uint8).reshape(-1)
        assert a.size <= self.n
        if a.size:
            ck(cu.cuMemcpyHtoD(self.ptr, a.ctypes.data, a.size))

    def put_i64(self, a: np.ndarray):
        self.put(np.ascontiguousarray(a, dtype=np.int64).view(np.uint8))

    def get(self, k=None) -> np.ndarray:
        k = self.n if k is None else k
        out = np.empty(k, np.uint8)
        if k:
            ck(cu.cuMemcpyDtoH(out.ctypes.data, self.ptr, k))
        return out

    def get_i64(self, count) -> np.ndarray:
        return self.get(8 * count).view(np.int64)

    def fill(self, v: int):
        if self.n:
            ck(cu.cuMemsetD8(self.ptr, v, self.n))

    def free(self):
        ck(cu.cuMemUnmap(self.va + self.gran, self.msz))
        ck(cu.cuMemRelease(self.h))
        ck(cu.cuMemAddressFree(self.va, self.vsz))

    @property
    def p(self):
        return ctypes.c_void_p(self.ptr)


def main():
    torch.cuda.init()
    torch.empty(1, device="cuda")  # the primary context is current from here on
    import paper_1910_05109_b200 as b64
    from paper_1910_05109_b200 import _lib

    L = _lib.lib()
    std = L.b64_alphabet_standard()
    url = L.b64_alphabet_url()
    V = ctypes.c_void_p
    info = torch.zeros(4, dtype=torch.int64, device="cuda")
    ip = info.data_ptr()
    ERR, ST, OLEN = V(ip), V(ip + 8), V(ip + 16)
    cases = 0

    def sync():
        torch.cuda.synchronize()

    def res():
        sync()
        v = info.tolist()
        return v[0], v[1] & 0xFFFFFFFF, v[2]  # the status is an int32 in the low half

    def G(n, where):
        return Guarded(n, where)

    wheres = ("tail", "head")
    # ---------------------------------------------------------------- single-stream encode / decode
    for n in (1, 2, 3, 4, 47, 767, 768, 769, 3001, 100_003, 600_001, 2_000_002):
        x = synth.data(n, seed=n)
        ref = oracle.encode(x)
        m = ref.size
        for wi in wheres:
            for wo in wheres:
                gi, go = G(n, wi), G(m, wo)
                gi.put(x)
                _lib.check(L.b64_encode(gi.p, n, go.p, std, None), "encode")
                sync()
                assert np.array_equal(go.get(), ref), ("encode", n, wi, wo)
                gi.free(), go.free()
                cases += 1
                # decode: text guarded, output guarded at its exact capacity 3*m/4
                gt, gd = G(m, wi), G(3 * (m // 4), wo)
                gt.put(ref)
                info.zero_()
                _lib.check(L.b64_decode_ex(gt.p, m, gd.p, std, ERR, ST, OLEN, None), "decode_ex")
                e, s, ol = res()
                assert e == -1 and ol == n and np.array_equal(gd.get(n), x), ("decode", n, wi, wo)
                # the same text with an error in its last quad
                t2 = ref.copy()
                t2[m - 3] = ord("*")
                gt.put(t2)
                info.zero_()
                _lib.check(L.b64_decode_ex(gt.p, m, gd.p, std, ERR, ST, OLEN, None), "decode_ex err")
                e, s, ol = res()
                assert e == oracle.decode(t2)[1], ("decode err", n, wi, wo, e)
                # chunk API, interior (no final quad)
                cell = torch.full((1,), b64.ERR_NONE, dtype=torch.int64, device="cuda")
                gt.put(ref)
                _lib.check(L.b64_decode_chunk(gt.p, m - 4, gd.p, std, 0, 0, V(cell.data_ptr()), None, None), "chunk")
                sync()
                assert int(cell.item()) == b64.ERR_NONE
                gt.free(), gd.free()
                cases += 3
    # ---------------------------------------------------------------- fused (context) decode, unpadded, lenient
    ctx = torch.empty(16, dtype=torch.uint8, device="cuda")
    _lib.check(L.b64_decode_ctx_init(V(ctx.data_ptr()), None), "ctx")
    for n in (600_001, 2_000_003):
        x = synth.data(n, seed=n)
        ref = oracle.encode(x)
        m = ref.size
        for w in wheres:
            gt, gd = G(m, w), G(3 * (m // 4), w)
            gt.put(ref)
            info.zero_()
            _lib.check(L.b64_decode_fused(gt.p, m, gd.p, std, ERR, ST, OLEN, V(ctx.data_ptr()), None), "fused")
            e, s, ol = res()
            assert e == -1 and ol == n and np.array_equal(gd.get(n), x)
            gt.free(), gd.free()
            cases += 1
    for n in (1, 2, 4, 5, 1000, 100_001):
        x = synth.data(n, seed=n + 9)
        tu = oracle.encode_unpadded(x, oracle.URL)
        m = tu.size
        cap = int(L.b64_decoded_len_max_unpadded(m))
        for w in wheres:
            gt, gd = G(m, w), G(cap, w)
            gt.put(tu)
            info.zero_()
            _lib.check(L.b64_decode_unpadded(gt.p, m, gd.p, url, ERR, ST, OLEN, None), "unpadded")
            e, s, ol = res()
            assert e == -1 and ol == n and np.array_equal(gd.get(n), x), ("unpadded", n, w)
            gt.free(), gd.free()
            cases += 1
    # ---------------------------------------------------------------- whitespace-skipping decode (all 3 paths)
    x = synth.data(700_000, seed=11)
    t = oracle.encode(x)
    mime = np.concatenate([np.concatenate([t[i: i + 76], np.frombuffer(b"\r\n", np.uint8)])
                           for i in range(0, t.size, 76)])
    for text in (mime[:7800], mime, np.concatenate([mime[:1000], [32], mime[1000:]]).astype(np.uint8)):
        m = text.size
        ref, rerr, _ = oracle.decode_ws(text)
        wsb = int(L.b64_decode_ws_workspace_bytes(m))
        for w in wheres:
            gt, gw = G(m, w), G(wsb, w)
            gd = G(3 * (m // 4), "head")  # d_out must be 16-byte aligned
            gt.put(text)
            info.zero_()
            _lib.check(L.b64_decode_ws(gt.p, m, gd.p, std, gw.p, wsb, ERR, ST, OLEN, None), "ws")
            e, s, ol = res()
            assert e == rerr and ol == ref.size and np.array_equal(gd.get(ol), ref), ("ws", m, w)
            gt.free(), gw.free(), gd.free()
            cases += 1
    # ---------------------------------------------------------------- batches + device offsets
    Ls = synth.loguniform_lengths(5000, hi=8192, seed=3)
    off = synth.offsets(Ls)
    x = synth.data(int(off[-1]), seed=3)
    eref, eoff = oracle.encode_batch(x, off)
    count = Ls.size
    for w in wheres:
        gx, goff, goo, gout = G(x.size, w), G(8 * (count + 1), w), G(8 * (count + 1), w), G(eref.size, w)
        gx.put(x)
        goff.put_i64(off)
        _lib.check(L.b64_encode_batch_offsets(goff.p, count, goo.p, None), "enc offsets")
        sync()
        assert np.array_equal(goo.get_i64(count + 1), eoff)
        _lib.check(L.b64_encode_batch(gx.p, goff.p, count, gout.p, goo.p, std, None), "enc batch")
        sync()
        assert np.array_equal(gout.get(), eref), ("enc batch", w)
        t = eref.copy()
        t[eoff[11] + 2] = ord("*")
        rout, roff, rst, rerr, rlen = oracle.decode_batch(t, eoff)
        gt, gdo, gdd = G(t.size, w), G(8 * (count + 1), w), G(int(roff[-1]), w)
        gt.put(t)
        _lib.check(L.b64_decode_batch_offsets(goo.p, count, gdo.p, None), "dec offsets")
        sync()
        assert np.array_equal(gdo.get_i64(count + 1), roff)
        gst, gerr, glen = G(4 * count, w), G(8 * count, w), G(8 * count, w)
        _lib.check(L.b64_decode_batch(gt.p, goo.p, count, gdd.p, gdo.p, std, gst.p, gerr.p, glen.p, None), "dec batch")
        sync()
        assert np.array_equal(gst.get(4 * count).view(np.int32), rst)
        assert np.array_equal(gerr.get_i64(count), rerr) and np.array_equal(glen.get_i64(count), rlen)
        for g in (gx, goff, goo, gout, gt, gdo, gdd, gst, gerr, glen):
            g.free()
        cases += 4
    # ---------------------------------------------------------------- streaming (pieces guarded one by one)
    x = synth.data(50_003, seed=5)
    ref = oracle.encode(x)
    carry = torch.zeros(8, dtype=torch.uint8, device="cuda")
    st = _lib.Stream()
    _lib.check(L.b64_encode_stream_begin(ctypes.byref(st), V(carry.data_ptr())), "es begin")
    got = []
    n_out = ctypes.c_int64(0)
    for a, b_ in ((0, 1), (1, 3), (3, 20_000), (20_000, 50_003)):
        gp = G(b_ - a, "tail")
        gp.put(x[a:b_])
        k = int(L.b64_stream_update_len(ctypes.byref(st), b_ - a))
        go = G(k, "tail")
        _lib.check(L.b64_encode_stream_update(ctypes.byref(st), gp.p, b_ - a, go.p, std, ctypes.byref(n_out), None), "esu")
        sync()
        got.append(go.get(n_out.value))
        gp.free(), go.free()
    go = G(int(L.b64_stream_end_len(ctypes.byref(st))), "tail")
    _lib.check(L.b64_encode_stream_end(ctypes.byref(st), go.p, std, ctypes.byref(n_out), None), "ese")
    sync()
    got.append(go.get(n_out.value))
    go.free()
    assert np.array_equal(np.concatenate(got), ref)
    cases += 1
    cell = torch.empty(1, dtype=torch.int64, device="cuda")
    st = _lib.Stream()
    _lib.check(L.b64_decode_stream_begin(ctypes.byref(st), V(carry.data_ptr()), V(cell.data_ptr()), None), "ds begin")
    got = []
    for a, b_ in ((0, 3), (3, 4), (4, 40_001), (40_001, ref.size)):
        gp = G(b_ - a, "tail")
        gp.put(ref[a:b_])
        k = int(L.b64_stream_update_len(ctypes.byref(st), b_ - a))
        go = G(k, "tail")
        _lib.check(L.b64_decode_stream_update(ctypes.byref(st), gp.p, b_ - a, go.p, std, ctypes.byref(n_out), None), "dsu")
        sync()
        got.append(go.get(n_out.value))
        gp.free(), go.free()
    go = G(int(L.b64_stream_end_len(ctypes.byref(st))), "tail")
    info.zero_()
    _lib.check(L.b64_decode_stream_end(ctypes.byref(st), go.p, std, ERR, ST, OLEN, ctypes.byref(n_out), None), "dse")
    e, s, ol = res()
    got.append(go.get(n_out.value))
    go.free()
    assert e == -1 and np.array_equal(np.concatenate(got)[: x.size], x)
    cases += 1
    # ---------------------------------------------------------------- grouped / fused codec launches
    xs = [synth.data(n, seed=n) for n in (300_003, 768 * 9, 5)]
    refs = [oracle.encode(v) for v in xs]
    gx = [G(v.size, "head") for v in xs]       # fast path: aligned starts
    ge = [G(r.size, "head") for r in refs]
    gt = [G(r.size, "head") for r in refs]
    gd = [G(3 * (r.size // 4), "head") for r in refs]
    for g, v in zip(gx, xs):
        g.put(v)
    for g, r in zip(gt, refs):
        g.put(r)
    k = len(xs)
    cells = torch.full((k,), b64.ERR_NONE, dtype=torch.int64, device="cuda")
    eitems = (_lib.EncodeItem * k)()
    ditems = (_lib.DecodeItem * k)()
    for i in range(k):
        eitems[i] = _lib.EncodeItem(gx[i].ptr, xs[i].size, ge[i].ptr, std)
        ditems[i] = _lib.DecodeItem(gt[i].ptr, refs[i].size, gd[i].ptr, std, 0, 1, 0, cells[i:].data_ptr())
    err = torch.empty(k, dtype=torch.int64, device="cuda")
    sts = torch.empty(k, dtype=torch.int32, device="cuda")
    ticket = torch.zeros(1, dtype=torch.int32, device="cuda")
    for rep in range(3):
        _lib.check(L.b64_codec_group_fused(eitems, k, ditems, k, V(err.data_ptr()), V(sts.data_ptr()),
                                           V(ticket.data_ptr()), None), "fused group")
        sync()
        assert err.tolist() == [-1] * k
        for i in range(k):
            assert np.array_equal(ge[i].get(), refs[i]) and np.array_equal(gd[i].get(xs[i].size), xs[i])
    cells.fill_(b64.ERR_NONE)
    _lib.check(L.b64_codec_group(eitems, k, ditems, k, None), "codec group")
    sync()
    assert cells.tolist() == [b64.ERR_NONE] * k
    for g in gx + ge + gt + gd:
        g.free()
    cases += 4
    # ---------------------------------------------------------------- host pipeline (device workspace guarded)
    n = 40_001
    x = synth.data(n, seed=8)
    ref = oracle.encode(x)
    wsb = int(L.b64_host_workspace_bytes(3072 * 2))
    gw = G(wsb, "tail")
    hx = torch.from_numpy(x).pin_memory()
    ho = torch.empty(ref.size, dtype=torch.uint8).pin_memory()
    _lib.check(L.b64_encode_host(V(hx.data_ptr()), n, V(ho.data_ptr()), std, gw.p, wsb, None, None, None), "eh")
    sync()
    assert np.array_equal(ho.numpy(), ref)
    ht = torch.from_numpy(ref.copy()).pin_memory()
    hy = torch.empty(3 * (ref.size // 4), dtype=torch.uint8).pin_memory()
    info.zero_()
    _lib.check(L.b64_decode_host(V(ht.data_ptr()), ref.size, V(hy.data_ptr()), std, gw.p, wsb, ERR, ST, OLEN,
                                 None, None, None), "dh")
    e, s, ol = res()
    assert e == -1 and ol == n and np.array_equal(hy.numpy()[:n], x)
    gw.free()
    cases += 2
    print(f"ALL OK {cases}", flush=True)


if __name__ == "__main__":
    main()
