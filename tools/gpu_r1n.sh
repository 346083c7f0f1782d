set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_full.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
tail -3 gpurun_out/pytest_gpu_full.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c3.json
timeout 600 python bench.py --workload c2x --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c2x.json
ls -la gpurun_out
