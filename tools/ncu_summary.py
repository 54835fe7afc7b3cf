"""Summarise an ncu --set full report: key roofline / pipe / stall metrics."""
import csv
import io
import subprocess
import sys

KEYS = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_bytes.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__grid_size',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'smsp__inst_executed.sum',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__cycles_elapsed.avg.per_second', 'smsp__issue_active.avg.pct_of_peak_sustained_active']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        for i, h in enumerate(hdr):
            if h in KEYS:
                print(f'{h:75s} {vals[i]:>22s} {units[i]}')
        stalls = [(float(vals[i]) if vals[i] not in ('', 'n/a') else 0.0, h) for i, h in enumerate(hdr)
                  if h.startswith('smsp__average_warp_latency_issue_stalled_') or
                  (h.startswith('smsp__warp_issue_stalled_') and h.endswith('_per_warp_active.pct'))]
        stalls.sort(reverse=True)
        for v, h in stalls[:8]:
            print(f'  stall {h:70s} {v:10.2f}')


if __name__ == '__main__':
    main(sys.argv[1])
