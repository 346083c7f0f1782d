# stackscan v5 (adaptive groups) + the full GPU tier + the default bench line + ncu.  Outputs in gpurun_out/.
mkdir -p gpurun_out /tmp/ncu
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee gpurun_out/smoke.txt
timeout 1500 python -m pytest -m gpu -x -q tests 2>&1 | tail -4 | tee gpurun_out/pytest_g.txt
timeout 1200 python bench.py 2>&1 | tail -1 > gpurun_out/bench_g.json
python -c "import json; d=json.load(open('gpurun_out/bench_g.json')); print(d['value'], d['e2e']['value'], d['e2e_api']['value'], d['kernel_ms'], d['roofline_stackscan']['frac'], d['parity'], {k: (v['value'], v['kernel_ms']) for k, v in d['extra'].items()})" | tee gpurun_out/g.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:upy_stackscan -s 1 -c 1 -o /tmp/ncu/stackscan -f \
  python bench.py --no-cpu --pyc 0 --no-extra --steps 1 --warmup 1 > gpurun_out/ncu_stackscan.log 2>&1
ncu -i /tmp/ncu/stackscan.ncu-rep --page raw --csv > gpurun_out/ncu_stackscan_raw.csv 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/traffic_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu --pyc 0 --no-extra \
  > gpurun_out/ncu_traffic.log 2>&1
