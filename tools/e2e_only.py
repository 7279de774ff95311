#!/usr/bin/env python3
"""A/B of the bench's end-to-end (host buffers) measurement: bench.e2e as is, and the same
HostPipeline step with fresh / reused pinned buffers and pipelines."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1910_05109_b200 as b64  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
cases = [bench.Case(b64, synth, torch, d, a, 1, 0, dev) for d in bench.LENGTH_DELTAS for a in ("std", "url")]
b64_bytes = sum(2 * c.m for c in cases)
keep = []


def bufs():
    hx = [torch.empty(c.n, dtype=torch.uint8, pin_memory=True) for c in cases]
    ht = [torch.empty(c.m, dtype=torch.uint8, pin_memory=True) for c in cases]
    hxo = [torch.empty(c.m, dtype=torch.uint8, pin_memory=True) for c in cases]
    hto = [torch.empty(max(c.mlen, 1), dtype=torch.uint8, pin_memory=True) for c in cases]
    for i, c in enumerate(cases):
        hx[i].copy_(c.x)
        ht[i].copy_(c.text)
    keep.append((hx, ht, hxo, hto))
    return hx, ht, hxo, hto


def measure(tag, pipe, hx, ht, hxo, hto, check=False):
    if check:
        for i, c in enumerate(cases):
            t = pipe.encode(hx[i], c.alpha, out=hxo[i])
            y, err = pipe.decode(ht[i], c.alpha, out=hto[i])
            if check == "equal":
                assert torch.equal(t, ht[i]) and torch.equal(y, hx[i])

    def step():
        for i, c in enumerate(cases):
            pipe.encode(hx[i], c.alpha, out=hxo[i], sync=False)
            pipe.decode(ht[i], c.alpha, out=hto[i], sync=False)
    step()
    pipe.join()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        step()
    pipe.join()
    e1.record()
    torch.cuda.synchronize()
    print(tag, round(b64_bytes / (e0.elapsed_time(e1) / 3 * 1e-3) / 1e9, 2), flush=True)


P = lambda: b64.HostPipeline(chunk_bytes=64 << 20)  # noqa: E731
measure("fresh bufs, fresh pipe", P(), *bufs())
measure("fresh bufs, fresh pipe, sync check first", P(), *bufs(), check=True)
b = bufs()
p = P()
measure("same bufs+pipe 1", p, *b)
measure("same bufs+pipe 2", p, *b)
measure("same bufs+pipe, check", p, *b, check=True)
measure("same bufs+pipe, check+equal", p, *b, check="equal")
measure("same bufs+pipe, after equal", p, *b)
measure("fresh, check+equal", P(), *bufs(), check="equal")
r = bench.e2e(b64, synth, torch, dev, argparse.Namespace(e2e_chunk_mib=64, e2e_steps=3), cases)
print("bench.e2e", r["value"], r["link"]["copies_only_same_pattern_gbs"])
