#!/bin/bash
# Profile the longest launch of a kernel: plain run, ncu launch list, then one `--set full`
# capture of that launch. Usage: tools/ncu_top.sh <tag> <kernel-regex> <cmd...>
# Outputs: gpurun_out/<tag>_plain.log, <tag>_launches.csv, <tag>.ncu-rep
set -u
TAG=$1; KRE=$2; shift 2
OUT=gpurun_out
"$@" > $OUT/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv "$@" > /dev/null 2>&1
IDX=$(python - "$OUT/${TAG}_launches.csv" "$KRE" <<'PY'
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
ki, vi = rows[h].index('Kernel Name'), rows[h].index('Metric Value')
ts = [float(r[vi].replace(',', '')) for r in rows[h + 1:] if len(r) > vi and re.search(sys.argv[2], r[ki])]
print(max(range(len(ts)), key=lambda i: ts[i]))
PY
)
echo "longest $KRE launch index: $IDX"
ncu --set full --clock-control none --import-source on -k regex:$KRE -s $IDX -c 1 -o $OUT/${TAG} "$@" > $OUT/${TAG}_ncu.log 2>&1
tail -1 $OUT/${TAG}_ncu.log
