mkdir -p gpurun_out/o1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/o1/pytest.log 2>&1; tail -3 gpurun_out/o1/pytest.log
for c in 4 3 2 1; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/o1/c$c.json 2> gpurun_out/o1/c$c.err
  echo "c$c: $(python tools/bench_summary.py < gpurun_out/o1/c$c.json)"; tail -1 gpurun_out/o1/c$c.err
done
