#!/bin/bash
# Round-2 measurement set: GPU tests, smoke, default bench (config 4, reference parity + CPU
# baseline), full-size parity of configs 2-5 against the reference. Outputs under gpurun_out/$1.
set -u
O=gpurun_out/${1:-r2}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1500 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 600 $O/bench_c4.json; echo
timeout 2400 python tools/parity_configs.py --out $O/parity > $O/parity.log 2>&1; tail -3 $O/parity.log
