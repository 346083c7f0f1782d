# stackscan v6 + decode 3.11 no-EXT path: parity + timing.  Outputs in gpurun_out/.
mkdir -p gpurun_out
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -m gpu -x -q tests/test_stackscan.py tests/test_decode.py tests/test_golden_gpu.py 2>&1 | tail -4 | tee gpurun_out/pytest_h.txt
timeout 900 python bench.py --no-cpu --pyc 0 --no-extra 2>&1 | tail -1 > gpurun_out/bench_h.json
python -c "import json; d=json.load(open('gpurun_out/bench_h.json')); print(d['kernel_ms'], d['roofline_decode']['frac'], d['roofline_stackscan']['ms'], d['roofline_stackscan']['frac'], d['parity'])" | tee gpurun_out/h.txt
timeout 900 python bench.py --workload c3_311 --no-cpu --pyc 0 --no-extra --steps 3 2>&1 | tail -1 > gpurun_out/bench_h311.json
python -c "import json; d=json.load(open('gpurun_out/bench_h311.json')); print('311', d['kernel_ms'], d['roofline_decode']['frac'], d['roofline_stackscan']['frac'], d['parity'])" | tee -a gpurun_out/h.txt
