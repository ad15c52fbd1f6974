#!/bin/bash
# Per-launch DRAM bytes, L2 hit rate, instructions and time of every MIH probe/piece launch of one
# untraced step (tools/one_step.py). Usage: tools/ncu_rounds.sh <tag> [config]  -> gpurun_out/<tag>_rounds.{csv,txt}
set -u
TAG=$1; C=${2:-4}; OUT=gpurun_out
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,lts__t_sectors_op_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:"mih_probe_kernel|mih_piece_kernel" --csv --log-file $OUT/${TAG}_rounds.csv \
    python tools/one_step.py --config $C > /dev/null 2>&1
python - "$OUT/${TAG}_rounds.csv" > $OUT/${TAG}_rounds.txt <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Metric Name' in r)
H = rows[h]
per = {}
for r in rows[h + 1:]:
    if len(r) < len(H): continue
    name, unit, val = r[H.index('Metric Name')], r[H.index('Metric Unit')], float(r[H.index('Metric Value')].replace(',', ''))
    scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'nsecond': 1e-6, 'usecond': 1e-3, 'msecond': 1, 'second': 1e3, 'ns': 1e-6, 'us': 1e-3, 'ms': 1, 's': 1e3}.get(unit, 1)
    d = per.setdefault(int(r[H.index('ID')]), {'k': r[H.index('Kernel Name')][:40]})
    d[name] = val * scale
tot = {}
print("id kernel ms dramGB l2hit% Minst issue% Ml2sect")
for i in sorted(per):
    d = per[i]
    gb = (d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)) / 1e9
    print(i, d['k'], round(d.get('gpu__time_duration.sum', 0), 3), round(gb, 3), round(d.get('lts__t_sector_hit_rate.pct', 0), 1),
          round(d.get('smsp__inst_executed.sum', 0) / 1e6, 1), round(d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0), 1),
          round(d.get('lts__t_sectors_op_read.sum', 0) / 1e6, 1))
    tot['ms'] = tot.get('ms', 0) + d.get('gpu__time_duration.sum', 0)
    tot['gb'] = tot.get('gb', 0) + gb
    tot['inst'] = tot.get('inst', 0) + d.get('smsp__inst_executed.sum', 0)
    tot['sect'] = tot.get('sect', 0) + d.get('lts__t_sectors_op_read.sum', 0)
print("total ms %.3f dramGB %.2f Ginst %.3f Gl2sect %.3f" % (tot['ms'], tot['gb'], tot['inst'] / 1e9, tot['sect'] / 1e9))
PY
cat $OUT/${TAG}_rounds.txt
