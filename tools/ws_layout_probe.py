#!/usr/bin/env python3
"""Whitespace decode of 1 GiB of data as MIME text: regular layout (one-pass line path) and
the same text with one stray blank at 1 KiB / the middle / near the end (the line pass stops
when it meets the break; then the general path runs).  CUDA events, L2 flushed."""
import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch, ctypes
import paper_1910_05109_b200 as b64, synth
dev = torch.device("cuda:0")
n = 1 << 30
x = synth.device_data(n, seed=0); t = b64.encode(x); m = t.numel()
lines = m // 76
body = t[: lines * 76].view(lines, 76)
crlf = torch.tensor([13, 10], dtype=torch.uint8, device=dev).expand(lines, 2)
tw = torch.cat([torch.cat([body, crlf], 1).reshape(-1), t[lines * 76:]])
out = torch.empty(3 * (m // 4) + 8, dtype=torch.uint8, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for tag, pos in (("regular", None), ("stray_at_1KiB", 1024), ("stray_mid", tw.numel() // 2),
                 ("stray_end", tw.numel() - 100), ("trailing_blank_lines", -1)):
    if pos == -1:
        tt = torch.cat([tw, torch.tensor([13, 10, 13, 10], dtype=torch.uint8, device=dev)])
    else:
        tt = tw if pos is None else torch.cat([tw[:pos], torch.tensor([32], dtype=torch.uint8, device=dev), tw[pos:]])
    ws = torch.empty(int(b64._lib.lib().b64_decode_ws_workspace_bytes(tt.numel())), dtype=torch.uint8, device=dev)
    o, err = b64.decode_ws(tt, out=out, workspace=ws)
    assert err == -1 and torch.equal(o, x)
    ts = []
    for k in range(8):
        flush.fill_(k)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); b64.decode_ws(tt, out=out, workspace=ws); b.record(); torch.cuda.synchronize()
        if k >= 3: ts.append(a.elapsed_time(b))
    print(tag, round(statistics.median(ts), 4))
