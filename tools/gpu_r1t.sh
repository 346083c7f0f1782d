set -x
mkdir -p gpurun_out
timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu --pyc 0 > gpurun_out/bench_c5.log 2>&1; tail -1 gpurun_out/bench_c5.log > gpurun_out/bench_c5.json
tail -5 gpurun_out/bench_c5.log
ls -la gpurun_out
