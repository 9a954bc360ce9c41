"""Summarise an ncu --set full report (raw page CSV) into the metrics that matter here."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum']
STALLS = ['long_scoreboard', 'mio_throttle', 'short_scoreboard', 'lg_throttle', 'selected', 'not_selected', 'wait',
          'math_pipe_throttle', 'barrier', 'membar', 'branch_resolving', 'no_instructions', 'dispatch_stall', 'sleeping']


def main(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    for d in data:
        print('-----', d[ix['Kernel Name']][:70])
        for w in WANT:
            if w in ix:
                print(f"  {w:66s} {d[ix[w]]:>14s} {units[ix[w]]}")
        st = []
        for s in STALLS:
            k = 'smsp__pcsamp_warps_issue_stalled_' + s
            if k in ix and d[ix[k]] not in ('', '0'):
                st.append((int(float(d[ix[k]].replace(',', ''))), s))
        st.sort(reverse=True)
        print('  stalls:', ', '.join(f'{s}={v}' for v, s in st[:8]))


if __name__ == '__main__':
    main(sys.argv[1])
