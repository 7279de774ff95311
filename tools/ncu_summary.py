#!/usr/bin/env python3
"""Summarise an ncu report (raw page) into the numbers DESIGN.md / profiles/ cite.
    python tools/ncu_summary.py gpurun_out/X_prof.ncu-rep [--json out.json]
"""
import csv, io, json, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__m_xbar2l1tex_read_bytes.sum', 'l1tex__m_l1tex2xbar_write_bytes.sum', 'lts__t_sectors.sum',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__cycles_elapsed.avg.per_second', 'dram__cycles_elapsed.avg.per_second']


def main():
    rep = sys.argv[1]
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for d in data:
        rec = {'kernel': d[hdr.index('Kernel Name')].split('(')[0]}
        for k in KEYS:
            if k in hdr:
                rec[k] = d[hdr.index(k)] + (' ' + units[hdr.index(k)] if units[hdr.index(k)] else '')
        st = [(h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), float(d[i] or 0))
              for i, h in enumerate(hdr) if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('per_issue_active.ratio')]
        rec['top_stalls_per_issue'] = {k: round(v, 3) for k, v in sorted(st, key=lambda t: -t[1])[:6]}
        rb = float(d[hdr.index('dram__bytes_read.sum')]) * (1e9 if 'Gbyte' in units[hdr.index('dram__bytes_read.sum')] else 1e6 if 'Mbyte' in units[hdr.index('dram__bytes_read.sum')] else 1)
        wb = float(d[hdr.index('dram__bytes_write.sum')]) * (1e9 if 'Gbyte' in units[hdr.index('dram__bytes_write.sum')] else 1e6 if 'Mbyte' in units[hdr.index('dram__bytes_write.sum')] else 1)
        rec['dram_bytes_total'] = rb + wb
        out.append(rec)
    for r in out:
        print('----', r['kernel'])
        for k, v in r.items():
            if k != 'kernel':
                print(f'  {k} = {v}')
    if '--json' in sys.argv:
        json.dump(out, open(sys.argv[sys.argv.index('--json') + 1], 'w'), indent=1)


if __name__ == '__main__':
    main()
