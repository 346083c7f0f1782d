# lean 3.11 decode: parity + timing.  Outputs in gpurun_out/.
mkdir -p gpurun_out
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -m gpu -x -q tests/test_decode.py tests/test_golden_gpu.py tests/test_stackscan.py 2>&1 | tail -4 | tee gpurun_out/pytest_i.txt
timeout 900 python bench.py --workload c3_311 --no-cpu --pyc 0 --no-extra --steps 3 2>&1 | tail -1 > gpurun_out/bench_i311.json
python -c "import json; d=json.load(open('gpurun_out/bench_i311.json')); print('311', d['kernel_ms'], d['roofline_decode']['frac'], d['parity'])" | tee gpurun_out/i.txt
timeout 600 ncu --set full --clock-control none -k regex:upy_decode -s 3 -c 1 --csv --page raw \
  python bench.py --workload c3_311 --no-cpu --pyc 0 --no-extra --steps 1 --warmup 2 > gpurun_out/ncu_decode311_lean_raw.csv 2>&1
