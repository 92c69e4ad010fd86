"""Summarise an ncu report (one kernel): time, throughputs, occupancy, stalls,
shared-memory wavefronts. python tools/ncu_summary.py REPORT.ncu-rep"""
import csv, io, subprocess, sys

def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    units = dict(zip(rows[0], rows[1]))  # ncu scales each metric's unit per report (ms/us, GB/MB, ...)
    return [dict(zip(rows[0], r), _units=units) for r in rows[2:]]

KEYS = ['gpu__time_duration.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed.avg.per_cycle_active', 'smsp__inst_executed.sum',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'smsp__inst_executed_op_shared_ld.sum', 'launch__occupancy_limit_shared_mem', 'launch__registers_per_thread',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'lts__t_sector_hit_rate.pct']

for d in raw(sys.argv[1]):
    print(d.get('Kernel Name', '')[:90])
    for k in KEYS:
        if k in d:
            print(f'  {k:70s} {d[k]} {d["_units"].get(k, "")}')
    st = {k: float(d[k]) for k in d if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')
          and d[k] not in ('', 'n/a')}
    for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]:
        print(f'  stall {k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]:30s} {v:.3f}')
