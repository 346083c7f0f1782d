# stack-scan kernel + 3.11 ring decode: parity, then the default bench line.  Outputs in gpurun_out/.
mkdir -p gpurun_out /tmp/ncu
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -m gpu -x -q tests/test_stackscan.py tests/test_decode.py tests/test_golden_gpu.py 2>&1 | tail -6 | tee gpurun_out/pytest_b.txt
timeout 1200 python bench.py --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench_b.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:upy_decode -s 3 -c 1 -o /tmp/ncu/decode311 -f \
  python bench.py --workload c3_311 --no-cpu --pyc 0 --no-extra --steps 1 --warmup 2 > gpurun_out/ncu_decode311.log 2>&1
ncu -i /tmp/ncu/decode311.ncu-rep --page raw --csv > gpurun_out/ncu_decode311_raw.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:upy_stackscan -s 1 -c 1 -o /tmp/ncu/stackscan -f \
  python bench.py --no-cpu --pyc 0 --no-extra --steps 1 --warmup 1 > gpurun_out/ncu_stackscan.log 2>&1
ncu -i /tmp/ncu/stackscan.ncu-rep --page raw --csv > gpurun_out/ncu_stackscan_raw.csv 2>&1
