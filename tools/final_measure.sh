#!/bin/bash
# Round-end measurement set (one gpurun call): tests, smoke, bench lines for every config / k /
# method, the reference CPU arm, ncu launch list of the default bench command, one --set full
# capture of the top probe launch and of the K7 tensor-core scan, and DRAM traffic per step.
# Outputs under gpurun_out/final/.
set -u
O=gpurun_out/final
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
b() { local tag=$1; shift; timeout 1200 python bench.py "$@" > $O/$tag.json 2> $O/$tag.err; python tools/bench_summary.py < $O/$tag.json | sed "s/^/$tag /"; }
b bench_c4 --config 4
for c in 1 2 3; do b bench_c$c --config $c; done
b bench_c5 --config 5 --no-cpu-baseline --steps 5
b bench_c4_k1 --config 4 --k 1 --no-cpu-baseline
b bench_c4_k1000 --config 4 --k 1000 --no-cpu-baseline
b bench_c2_k1 --config 2 --k 1 --no-cpu-baseline
b bench_c2_k100 --config 2 --k 100 --no-cpu-baseline
for c in 3 4 5; do b scan_c$c --config $c --method scan --no-cpu-baseline --steps 5; done
b ref_c4 --impl reference
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_c4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launches_bench_c4.log 2>&1
python tools/launch_summary.py $O/launches_bench_c4.csv > $O/launches_bench_c4_summary.csv
head -8 $O/launches_bench_c4_summary.csv
timeout 1500 bash tools/ncu_top.sh final/c4_probe mih_probe_kernel python tools/one_step.py --config 4
python tools/ncu_summary.py $O/c4_probe.ncu-rep > $O/ncu_full_c4_probe.txt 2>&1
python tools/ncu_mem_sites.py $O/c4_probe.ncu-rep > $O/ncu_mem_sites_c4_probe.txt 2>&1
timeout 900 bash tools/ncu_top.sh final/k7_256 tc_scan_kernel python tools/bench_tcscan.py 2e7 256 10000 100 tc
python tools/ncu_summary.py $O/k7_256.ncu-rep > $O/ncu_full_k7_256.txt 2>&1
for c in 4 3 2; do timeout 1200 bash tools/ncu_traffic.sh $c > $O/traffic_c$c.json 2>&1; cat $O/traffic_c$c.json; done
