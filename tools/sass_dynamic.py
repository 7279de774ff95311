#!/usr/bin/env python3
"""Dynamic instruction mix of the hot loop of each kernel in an ncu report (`--page source`,
SASS view, 'Instructions Executed' per instruction): the instructions executed exactly as
often as the loop trips (the modal execution count among the heavy ones) form the hot path;
printed with their opcode mix and the warp-instructions per 64 base64 chars.

    python tools/sass_dynamic.py REPORT KERNEL_REGEX CHARS_PER_TRIP [label]

CHARS_PER_TRIP: base64 chars one warp handles per loop trip (1024 for the fast kernels' chunk).
"""
import collections
import csv
import io
import subprocess
import sys

rep, k, cpt = sys.argv[1], sys.argv[2], int(sys.argv[3])
label = sys.argv[4] if len(sys.argv) > 4 else k
raw = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '-k', k, '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
sections, cur = [], None
for r in rows:
    if r and r[0] == 'Kernel Name':
        cur = {'name': r[1], 'rows': []}
        sections.append(cur)
    elif cur is not None and r and r[0] == 'Address':
        cur['hdr'] = r
    elif cur is not None and 'hdr' in cur and len(r) == len(cur['hdr']) and r[2].isdigit():
        cur['rows'].append(dict(zip(cur['hdr'], r)))
if not sections:
    sys.exit(f'no kernel matching {k}')
sec = sections[0]
E = 'Instructions Executed'
data = sec['rows']
total = sum(int(d[E] or 0) for d in data)
counts = collections.Counter(int(d[E] or 0) for d in data if int(d[E] or 0) > 0)
# the loop trip count: the execution count that carries the most executed instructions
trip, _ = max(counts.items(), key=lambda kv: kv[0] * kv[1])
hot = [d for d in data if int(d[E] or 0) == trip]
ops = collections.Counter()
for d in hot:
    src = d['Source'].strip()
    toks = src.split()
    op = toks[1] if toks[0].startswith('@') else toks[0]
    ops[op] += 1
print(f'## {label}: {sec["name"][:100]}')
print(f'   warp-instructions executed: {total:,}; hot path: {len(hot)} instructions x {trip:,} trips '
      f'({len(hot) * trip / total:.0%} of all)')
print(f'   hot path per trip ({cpt} chars per warp): {len(hot)} warp-instructions = {len(hot) / cpt * 64:.2f} per 64 chars; '
      f'whole kernel: {total / (trip * cpt / 64):.2f} per 64 chars')
print('   mix: ' + ', '.join(f'{o} {c}' for o, c in ops.most_common()))
