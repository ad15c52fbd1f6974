#!/bin/bash
# Round-2 measurement set (one gpurun call): GPU tests, smoke, bench lines for every config / k /
# method (config 4 = the default line, with the reference's CPU MIH + scan baseline and the
# reference-parity gate), the reference CPU arm, a torchrun (NCCL) line, the ncu launch list of
# the default bench command, --set full captures of the top MIH probe launch and of the K7
# tensor-core scan, and DRAM traffic per step. Outputs under gpurun_out/$1 (default r2final).
set -u
O=gpurun_out/${1:-r2final}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
b() { local tag=$1; shift; timeout 1500 python bench.py "$@" > $O/$tag.json 2> $O/$tag.err; python tools/bench_summary.py < $O/$tag.json | sed "s/^/$tag /"; }
b bench_c4 --config 4
for c in 1 2 3 5; do b bench_c$c --config $c; done
b bench_c4_k1 --config 4 --k 1 --no-cpu-baseline
b bench_c4_k1000 --config 4 --k 1000 --no-cpu-baseline
b bench_c2_k1 --config 2 --k 1 --no-cpu-baseline
b bench_c2_k100 --config 2 --k 100 --no-cpu-baseline
for c in 3 4 5; do b scan_c$c --config $c --method scan --no-cpu-baseline --steps 5; done
b ref_c4 --impl reference
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --config 3 --no-cpu-baseline --steps 5 > $O/torchrun1_c3.json 2> $O/torchrun1_c3.err
python tools/bench_summary.py < $O/torchrun1_c3.json | sed "s/^/torchrun1_c3 /"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_c4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launches_bench_c4.log 2>&1
python tools/launch_summary.py $O/launches_bench_c4.csv > $O/launches_bench_c4_summary.csv
head -8 $O/launches_bench_c4_summary.csv
timeout 1500 bash tools/ncu_top.sh ${1:-r2final}/c4_probe mih_probe_kernel python tools/one_step.py --config 4
python tools/ncu_summary.py $O/c4_probe.ncu-rep > $O/ncu_full_c4_probe.txt 2>&1
python tools/ncu_mem_sites.py $O/c4_probe.ncu-rep 25 > $O/ncu_mem_sites_c4_probe.txt 2>&1
python tools/ncu_src_lines.py $O/c4_probe.ncu-rep 40 > $O/ncu_src_lines_c4_probe.txt 2>&1
timeout 900 bash tools/ncu_rounds.sh ${1:-r2final}/c4 4 > /dev/null 2>&1
timeout 900 bash tools/ncu_top.sh ${1:-r2final}/k7_256 tc_scan_kernel python tools/bench_tcscan.py 4e8 256 10000 100 tc
python tools/ncu_summary.py $O/k7_256.ncu-rep > $O/ncu_full_k7_256.txt 2>&1
for c in 4 3 2; do timeout 1200 bash tools/ncu_traffic.sh $c > $O/traffic_c$c.json 2>&1; mv gpurun_out/traffic_c$c.* $O/ 2>/dev/null; tail -1 $O/traffic_c$c.json; done
