# stackscan v3 parity/timing; hoist variant A/B (same session).  Outputs in gpurun_out/.
mkdir -p gpurun_out
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -m gpu -x -q tests/test_stackscan.py tests/test_golden_gpu.py 2>&1 | tail -4 | tee gpurun_out/pytest_d.txt
for v in base hoist base hoist; do
  if [ $v = base ]; then L=; else L=paper_2403_13839_b200/_variants/$v.so; fi
  UPY_LIB=$L timeout 900 python bench.py --no-cpu --pyc 0 --no-extra 2>&1 | tail -1 > gpurun_out/bench_d_$v.json
  python -c "import json; d=json.load(open('gpurun_out/bench_d_$v.json')); print('$v', d['kernel_ms'], d['roofline_stackscan']['ms'], d['roofline_stackscan']['frac'], d['parity'])" | tee -a gpurun_out/ab_d.txt
done
