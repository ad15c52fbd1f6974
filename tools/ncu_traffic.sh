#!/bin/bash
# DRAM traffic of every MIH probe/piece launch of ONE untraced step of a bench config, plus the
# algorithmic bytes of that step. Usage: tools/ncu_traffic.sh <config>  -> gpurun_out/traffic_c<config>.*
set -u
C=$1; OUT=gpurun_out
python tools/one_step.py --config $C > $OUT/traffic_c${C}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
python tools/one_step.py --config $C --traced > $OUT/traffic_c${C}_alg.json 2>/dev/null
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"mih_probe_kernel|mih_piece_kernel" --csv --log-file $OUT/traffic_c${C}.csv \
    python tools/one_step.py --config $C > /dev/null 2>&1
python - "$OUT/traffic_c${C}.csv" "$OUT/traffic_c${C}_alg.json" <<'PY'
import csv, json, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Metric Name' in r)
H = rows[h]
tot = {}
launches = set()
for r in rows[h + 1:]:
    if len(r) < len(H): continue
    name, unit, val = r[H.index('Metric Name')], r[H.index('Metric Unit')], float(r[H.index('Metric Value')].replace(',', ''))
    scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'nsecond': 1e-9, 'usecond': 1e-6, 'msecond': 1e-3, 'second': 1}.get(unit, 1)
    tot[name] = tot.get(name, 0) + val * scale
    launches.add(r[H.index('ID')])
alg = json.load(open(sys.argv[2]))
traffic = tot.get('dram__bytes_read.sum', 0) + tot.get('dram__bytes_write.sum', 0)
print(json.dumps({"config": alg["config"], "launches": len(launches), "dram_bytes_per_step": traffic,
                  "alg_bytes_per_step": alg["alg_bytes_per_step"], "traffic_over_alg": traffic / alg["alg_bytes_per_step"],
                  "kernel_time_s_serialised": tot.get('gpu__time_duration.sum', 0)}))
PY
