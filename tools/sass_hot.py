#!/usr/bin/env python3
"""Per-instruction stall samples of one kernel in an ncu report (--page source, SASS view):
the hottest instructions and the sample share of basic regions.
    python tools/sass_hot.py REPORT KERNEL_REGEX [top]"""
import csv, io, subprocess, sys

rep, k = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '-k', k, '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[2].isdigit()]
n_kern = sum(1 for r in rows if r and r[0] == 'Kernel Name')
S = 'Warp Stall Sampling (All Samples)'
E = 'Instructions Executed'
tot = sum(int(d[S] or 0) for d in data)
tot_i = sum(int(d[E] or 0) for d in data)
print(f'{n_kern} kernel section(s); {len(data)} SASS instructions, {tot} stall samples, {tot_i} warp-instructions executed')
for i, d in enumerate(data):
    d['_i'] = i
for d in sorted(data, key=lambda d: -int(d[S] or 0))[:top]:
    print(f"{d['_i']:5d} {int(d[S] or 0)/tot*100:6.2f}% exec={d[E]:>10} {d['Source'].strip()[:90]}")
