mkdir -p gpurun_out/g1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g1/pytest.log 2>&1; tail -3 gpurun_out/g1/pytest.log
for v in "" _g4 _g3; do
  L=$PWD/paper_1307_2982_b200/libmihg$v.so
  MIHG_LIB_PATH=$L timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/g1/c4$v.json 2> gpurun_out/g1/c4$v.err
  echo "lib$v: $(python tools/bench_summary.py < gpurun_out/g1/c4$v.json)"; tail -2 gpurun_out/g1/c4$v.err
done
MIHG_GROUP_PROBE=0 timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/g1/c4_old.json 2> gpurun_out/g1/c4_old.err
echo "old: $(python tools/bench_summary.py < gpurun_out/g1/c4_old.json)"
