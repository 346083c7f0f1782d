# stackscan v4 (TMA stage) parity + timing; decode (tma.h refactor) parity.  Outputs in gpurun_out/.
mkdir -p gpurun_out
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -m gpu -x -q tests/test_stackscan.py tests/test_decode.py 2>&1 | tail -4 | tee gpurun_out/pytest_f.txt
timeout 900 python bench.py --no-cpu --pyc 0 --no-extra 2>&1 | tail -1 > gpurun_out/bench_f.json
python -c "import json; d=json.load(open('gpurun_out/bench_f.json')); print(d['kernel_ms'], d['roofline_stackscan'], d['parity'])" | tee gpurun_out/f.txt
timeout 900 python bench.py --workload c4 --no-cpu --pyc 0 --steps 1 --warmup 1 2>&1 | tail -1 > gpurun_out/bench_f_c4.json
python -c "import json; d=json.load(open('gpurun_out/bench_f_c4.json')); print(d['roofline_stackscan'])" | tee -a gpurun_out/f.txt
