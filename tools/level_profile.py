"""Per-launch table of one NR refactorisation from an ncu CSV launch list
(factor levels, tail-level classes, dense tail), with section totals.

    ACPF_NR_DEVLOOP=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,\
sm__inst_executed.avg.per_cycle_active --clock-control none -k regex:"nr_factor|nr_tail" --csv \
--log-file levels.csv python tools/step_probe.py 65536 1
    python tools/level_profile.py levels.csv
"""
import collections
import csv
import sys

SCALE_T = {'ns': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'msecond': 1.0, 'ms': 1.0, 'nsecond': 1e-6}
SCALE_B = {'byte': 1e-9, 'Kbyte': 1e-6, 'Mbyte': 1e-3, 'Gbyte': 1.0}

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
launches = collections.OrderedDict()
for r in rows:
    d = launches.setdefault(int(r[0]), {'name': r[4], 'grid': int(r[8].strip('()').split(',')[0])})
    d[r[12]] = (float(r[14].replace(',', '')), r[13])
seq = list(launches.values())
tails = [i for i, d in enumerate(seq) if 'nr_tail' in d['name']]
start, end = tails[0] + 1, tails[1] + 1  # the second refactorisation (warm L2/TLB)
ms = lambda d: d['gpu__time_duration.sum'][0] * SCALE_T[d['gpu__time_duration.sum'][1]]
gb = lambda d, k: d[k][0] * SCALE_B[d[k][1]]
m = lambda d, k: d[k][0]
sect = collections.OrderedDict((k, [0.0, 0.0, 0]) for k in ('sparse levels', 'tail-level classes', 'dense tail'))
print(f"{'#':>3} {'kernel':12s} {'CTAs':>7} {'ms':>7} {'rd GB':>6} {'wr GB':>6} {'L2 hit':>6} {'warps%':>6} {'IPC':>5}")
for i in range(start, end):
    d = seq[i]
    name = 'tail' if 'nr_tail' in d['name'] else 'factor'
    t = ms(d)
    rd, wr = gb(d, 'dram__bytes_read.sum'), gb(d, 'dram__bytes_write.sum')
    print(f"{i - start:3d} {name:12s} {d['grid']:7d} {t:7.3f} {rd:6.2f} {wr:6.2f} {m(d, 'lts__t_sector_hit_rate.pct'):6.1f} "
          f"{m(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} {m(d, 'sm__inst_executed.avg.per_cycle_active'):5.2f}")
    seq[i]['_t'], seq[i]['_b'] = t, rd + wr
n_cls = int(sys.argv[2]) if len(sys.argv) > 2 else 4  # tail-level classes: the launches before the dense tail
for i in range(start, end):
    d = seq[i]
    k = 'dense tail' if 'nr_tail' in d['name'] else ('tail-level classes' if i >= end - 1 - n_cls else 'sparse levels')
    sect[k][0] += d['_t']
    sect[k][1] += d['_b']
    sect[k][2] += 1
tot = sum(v[0] for v in sect.values())
print(f"one refactorisation (launch list, serialised, cold per launch): {tot:.2f} ms")
for k, (t, b, n) in sect.items():
    print(f"  {k:20s} {n:3d} launches {t:7.2f} ms ({t / tot:5.1%})  DRAM {b:6.1f} GB")
