#!/usr/bin/env python
"""Summarise an ncu report (raw page): duration, DRAM, pipes, issue, stall reasons."""
import csv, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'sm__cycles_elapsed.avg.per_second', 'dram__bytes_read.sum',
        'dram__bytes_write.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__inst_executed.sum', 'sm__inst_executed.avg.per_cycle_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'lts__t_bytes.sum', 'smsp__cycles_active.avg.pct_of_peak_sustained_elapsed']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}
        print('kernel:', d.get('Kernel Name', ('?',))[0][:90])
        for k in KEYS:
            if k in d:
                print(f'  {k:70s} {d[k][0]:>16s} {d[k][1]}')
        st = []
        for k, (v, u) in d.items():
            if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued'):
                try:
                    st.append((float(v.replace(',', '')), k))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        print('  stall samples (top):')
        for v, k in sorted(st, reverse=True)[:10]:
            print(f'    {k.replace("smsp__pcsamp_warps_issue_stalled_", ""):30s} {v:8.0f} {100 * v / tot:5.1f}%')


if __name__ == '__main__':
    for p in sys.argv[1:]:
        main(p)
