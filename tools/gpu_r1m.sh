# double-buffered e2e; pyc fetch buffer reuse
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c3.json
timeout 600 python bench.py --workload c3_311 --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c3_311.json
ls -la gpurun_out
