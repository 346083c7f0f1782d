# stack-scan v2 (descriptor table) parity + timing; decode 3.11 source profile.  Outputs in gpurun_out/.
mkdir -p gpurun_out /tmp/ncu
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -m gpu -x -q tests/test_stackscan.py 2>&1 | tail -4 | tee gpurun_out/pytest_c.txt
timeout 900 python bench.py --no-cpu --pyc 0 --no-extra 2>&1 | tail -1 | tee gpurun_out/bench_c.json
timeout 900 python bench.py --workload c4 --no-cpu --pyc 0 --steps 2 --warmup 1 2>&1 | tail -1 | tee gpurun_out/bench_c4.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:upy_stackscan -s 1 -c 1 -o /tmp/ncu/stackscan -f \
  python bench.py --no-cpu --pyc 0 --no-extra --steps 1 --warmup 1 > gpurun_out/ncu_stackscan.log 2>&1
ncu -i /tmp/ncu/stackscan.ncu-rep --page raw --csv > gpurun_out/ncu_stackscan_raw.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:upy_decode -s 3 -c 1 -o /tmp/ncu/decode311 -f \
  python bench.py --workload c3_311 --no-cpu --pyc 0 --no-extra --steps 1 --warmup 2 > gpurun_out/ncu_decode311.log 2>&1
ncu -i /tmp/ncu/decode311.ncu-rep --page source --csv > /tmp/ncu/decode311_source.csv 2>&1
gzip -c /tmp/ncu/decode311_source.csv > gpurun_out/ncu_decode311_source.csv.gz
