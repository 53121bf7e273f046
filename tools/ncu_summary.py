#!/usr/bin/env python3
"""Per-kernel summary of an ncu report: time, DRAM bytes, pipe utilisation,
occupancy and the top stall reasons.   python tools/ncu_summary.py rep.ncu-rep"""
import csv, io, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'smsp__inst_executed.sum',
        'launch__registers_per_thread', 'launch__grid_size', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__inst_executed_pipe_fp64.sum', 'sm__inst_executed_pipe_fp64.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']


def main():
    out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    for r in data:
        print('==', r[hdr.index('Kernel Name')][:70])
        vals = []
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                short = k.replace('sm__', '').replace('smsp__', '').replace('.avg.pct_of_peak_sustained_active', '%').replace('.sum', '')
                vals.append(f"{short}={r[i]}{units[i] if units[i] not in ('%', '') else ''}")
        print('   ' + '  '.join(vals))
        st = [(h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), float(r[i]))
              for i, h in enumerate(hdr) if h.startswith('smsp__average_warps_issue_stalled_')
              and h.endswith('_per_issue_active.ratio') and r[i] not in ('', 'n/a')]
        st.sort(key=lambda x: -x[1])
        print('   stalls ' + ', '.join(f'{a}={b:.2f}' for a, b in st[:7]))


if __name__ == '__main__':
    main()
