# 3.11 warp decode validation: decode-record parity test + full GPU suite + 3.11 benches
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --durations=5 -p no:cacheprovider > gpurun_out/pytest_gpu_full.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
tail -12 gpurun_out/pytest_gpu_full.txt
timeout 600 python bench.py --workload c3_311 --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_c3_311.json
timeout 300 python bench.py --workload c2_311 --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_c2_311.json
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_c3.json
ls -la gpurun_out
