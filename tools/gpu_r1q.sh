# StepCtx by value into step (argval reads in registers)
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_full.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
tail -3 gpurun_out/pytest_gpu_full.txt
for r in 1 2; do timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_c3_$r.json; done
timeout 300 python bench.py --workload c3_311 --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_c3_311.json
ls -la gpurun_out
