#!/usr/bin/env python3
"""Where does the end-to-end (host buffers) step lose against the PCIe link?

Times, for the bench's configs[1] cases (6 x 64 MiB (+0/1/2), std/url):
  * pipe_<chunk>: the bench's e2e step through b64.HostPipeline at several chunk sizes;
  * copies_only: the same H2D / D2H byte streams with no kernels, issued the same way
    (H2D of call i after D2H of call i-2, two staging areas), i.e. the pattern's ceiling;
  * duplex: one 256 MiB H2D and one 256 MiB D2H concurrently.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1910_05109_b200 as b64  # noqa: E402
import synth  # noqa: E402


def ev_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    N = 64 << 20
    cases = []
    for d in (0, 1, 2):
        for al in (b64.standard(), b64.url()):
            x = synth.device_data(N + d, seed=0)
            t = b64.encode(x, al)
            hx = torch.empty(x.numel(), dtype=torch.uint8, pin_memory=True)
            ht = torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True)
            hx.copy_(x)
            ht.copy_(t)
            cases.append((al, hx, ht, torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True),
                          torch.empty(3 * (t.numel() // 4), dtype=torch.uint8, pin_memory=True)))
    b64_bytes = sum(2 * c[2].numel() for c in cases)
    res = {}
    for mib in (16, 32, 64, 96, 128):
        pipe = b64.HostPipeline(chunk_bytes=mib << 20)

        def step():
            for al, hx, ht, hxo, hto in cases:
                pipe.encode(hx, al, out=hxo, sync=False)
                pipe.decode(ht, al, out=hto, sync=False)
            pipe.join()

        ms = ev_time(step)
        res[f"pipe_{mib}MiB"] = round(b64_bytes / (ms * 1e-3) / 1e9, 2)
        del pipe
    # copies only, same pattern
    dev = torch.device("cuda", 0)
    stage = [torch.empty(200 << 20, dtype=torch.uint8, device=dev) for _ in range(2)]
    sh, sd = torch.cuda.Stream(), torch.cuda.Stream()
    done = [None, None]

    def copies():
        k = 0
        cur = torch.cuda.current_stream()
        sh.wait_stream(cur)
        sd.wait_stream(cur)
        for al, hx, ht, hxo, hto in cases:
            for src, dst in ((hx, hxo), (ht, hto)):
                w = k & 1
                k += 1
                if done[w] is not None:
                    sh.wait_event(done[w])
                with torch.cuda.stream(sh):
                    stage[w][: src.numel()].copy_(src, non_blocking=True)
                e = torch.cuda.Event()
                e.record(sh)
                sd.wait_event(e)
                with torch.cuda.stream(sd):
                    dst.copy_(stage[w][: dst.numel()], non_blocking=True)
                d = torch.cuda.Event()
                d.record(sd)
                done[w] = d
        cur.wait_stream(sh)
        cur.wait_stream(sd)

    ms = ev_time(copies)
    res["copies_only_same_pattern"] = round(b64_bytes / (ms * 1e-3) / 1e9, 2)
    hb = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
    hb2 = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
    db, db2 = torch.empty_like(hb, device=dev), torch.empty_like(hb, device=dev)

    def duplex():
        cur = torch.cuda.current_stream()
        sh.wait_stream(cur)
        sd.wait_stream(cur)
        with torch.cuda.stream(sh):
            db.copy_(hb, non_blocking=True)
        with torch.cuda.stream(sd):
            hb2.copy_(db2, non_blocking=True)
        cur.wait_stream(sh)
        cur.wait_stream(sd)

    ms = ev_time(duplex)
    res["duplex_each_way_gbs"] = round((256 << 20) / (ms * 1e-3) / 1e9, 2)
    res["h2d_gbs"] = round((256 << 20) / (ev_time(lambda: db.copy_(hb, non_blocking=True)) * 1e-3) / 1e9, 2)
    res["d2h_gbs"] = round((256 << 20) / (ev_time(lambda: hb2.copy_(db2, non_blocking=True)) * 1e-3) / 1e9, 2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
