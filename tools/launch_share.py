#!/usr/bin/env python3
"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel name.
    python tools/launch_share.py gpurun_out/r1_launches.csv
Per-launch times under ncu are cold-cache and serialised: compare SHARES of the
codec step, not absolute times."""
import csv
import sys
from collections import defaultdict


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
    hdr_like = {"Kernel Name": 4, "Metric Value": 14}
    by = defaultdict(list)
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "")
        by[name].append(float(r[14]))
    codec = {k: v for k, v in by.items() if k.startswith("b64::")}
    tot_codec = sum(sum(v) for v in codec.values())
    print(f"{'kernel':60s} {'launches':>8s} {'mean_us':>9s} {'share_of_codec':>15s}")
    for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
        share = f"{100 * sum(v) / tot_codec:14.1f}%" if k in codec else ""
        print(f"{k[:60]:60s} {len(v):8d} {sum(v) / len(v) / 1e3:9.2f} {share:>15s}")


if __name__ == "__main__":
    main()
