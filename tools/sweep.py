#!/usr/bin/env python3
"""Size sweep of the fast encode / decode paths (one process = one kernel variant,
selected by the B64_* environment variables).  Prints one JSON line per size:
median op time with L2 flushed before each rep, base64 GB/s and HBM traffic GB/s,
next to a D2D copy of the same base64 byte count.

    B64_DEC_DEPTH=2 python tools/sweep.py --sizes 16M,64M,256M,1G
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1910_05109_b200 as b64  # noqa: E402
import synth  # noqa: E402


def parse_size(s):
    mult = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}
    return int(float(s[:-1]) * mult[s[-1]]) if s[-1] in mult else int(s)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--sizes", default="1M,4M,16M,64M,256M,1G")
    p.add_argument("--reps", type=int, default=20)
    p.add_argument("--tag", default=os.environ.get("B64_TAG", ""))
    p.add_argument("--group", type=int, default=0, help="also time k grouped streams of each size (one launch)")
    p.add_argument("--batch", type=int, default=0, help="time configs[3]-style batches of this many strings instead")
    p.add_argument("--batch-len", type=int, default=0, help="with --batch: every string this long (else log-uniform)")
    a = p.parse_args()
    dev = torch.device("cuda:0")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_r = torch.zeros(64 << 20, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    def timed(fn, reps):
        evs = []
        for k in range(reps + 3):
            flush.fill_(k & 255)
            flush_r.sum()
            torch.cuda._sleep(200_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        return statistics.median([e0.elapsed_time(e1) for e0, e1 in evs[3:]])

    if a.batch:  # log-uniform string lengths in [1, 64 KiB] (configs[3] recipe)
        import numpy as np

        Ls = (np.full(a.batch, a.batch_len, dtype=np.int64) if a.batch_len
              else synth.loguniform_lengths(a.batch, seed=0))
        off = synth.offsets(Ls)
        x = synth.device_data(int(off[-1]), seed=0)
        doff = torch.from_numpy(off).to(dev)
        enc, eoff = b64.encode_batch(x, doff)
        tot_in, tot_out = int(off[-1]), int(eoff[-1].item())
        lens = eoff[1:] - eoff[:-1]
        doo = torch.zeros(len(Ls) + 1, dtype=torch.int64, device=dev)
        torch.cumsum(3 * torch.div(lens, 4, rounding_mode="floor"), 0, out=doo[1:])
        dout = torch.empty(int(doo[-1].item()) + 16, dtype=torch.uint8, device=dev)
        te = timed(lambda: b64.encode_batch(x, doff, out=enc, out_off=eoff), a.reps)
        td = timed(lambda: b64.decode_batch(enc, eoff, out=dout, out_off=doo), a.reps)
        print(json.dumps({"tag": a.tag, "batch": a.batch, "len": a.batch_len, "in": tot_in, "b64": tot_out,
                          "enc": {"us": round(te * 1e3, 1), "traffic_gbs": round((tot_in + tot_out) / te / 1e6, 1)},
                          "dec": {"us": round(td * 1e3, 1), "traffic_gbs": round((tot_in + tot_out) / td / 1e6, 1)}}),
              flush=True)
        return
    for s in a.sizes.split(","):
        n = parse_size(s)
        x = synth.device_data(n, seed=0)
        t = b64.encode(x)
        o = torch.empty(3 * (t.numel() // 4), dtype=torch.uint8, device=dev)
        cell = torch.empty(1, dtype=torch.int64, device=dev)
        d = torch.empty_like(t)
        res = {"tag": a.tag, "n": n, "m": t.numel()}
        for name, fn in (("enc", lambda: b64.encode(x, out=t)),
                         ("dec", lambda: b64.decode_chunk(t, 0, True, cell, out=o)),
                         ("copy", lambda: d.copy_(t))):
            evs = []
            for k in range(a.reps + 3):
                flush.fill_(k & 255)
                flush_r.sum()
                torch.cuda._sleep(200_000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn()
                e1.record(stream)
                evs.append((e0, e1))
            torch.cuda.synchronize()
            ms = statistics.median([e0.elapsed_time(e1) for e0, e1 in evs[3:]])
            traffic = {"enc": n + t.numel(), "dec": t.numel() + n, "copy": 2 * t.numel()}[name]
            res[name] = {"us": round(ms * 1e3, 2), "b64_gbs": round(t.numel() / ms / 1e6, 1),
                         "traffic_gbs": round(traffic / ms / 1e6, 1)}
        if a.group:
            xs = [synth.device_data(n + (i % 3), seed=0) for i in range(a.group)]
            ts = b64.encode_group(xs)
            cells = torch.full((a.group,), b64.ERR_NONE, dtype=torch.int64, device=dev)
            outs = [torch.empty(3 * (tt.numel() // 4), dtype=torch.uint8, device=dev) for tt in ts]
            tot_n = sum(xx.numel() for xx in xs)
            tot_m = sum(tt.numel() for tt in ts)
            for name, fn in (("genc", lambda: b64.encode_group(xs, outs=ts)),
                             ("gdec", lambda: b64.decode_group(ts, outs=outs, cells=cells))):
                evs = []
                for k in range(a.reps + 3):
                    flush.fill_(k & 255)
                    flush_r.sum()
                    torch.cuda._sleep(200_000)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    fn()
                    e1.record(stream)
                    evs.append((e0, e1))
                torch.cuda.synchronize()
                ms = statistics.median([e0.elapsed_time(e1) for e0, e1 in evs[3:]])
                res[name] = {"us": round(ms * 1e3, 2), "traffic_gbs": round((tot_n + tot_m) / ms / 1e6, 1)}
            del xs, ts, outs
        print(json.dumps(res), flush=True)
        del x, t, o, d
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
