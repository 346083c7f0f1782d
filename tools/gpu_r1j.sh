# 3.11 parallel decode (pass-1 scan), fast-path guard, __ldg opcode table, L1 carveout; allocnoinl variant
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --durations=5 -p no:cacheprovider > gpurun_out/pytest_gpu_full.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
tail -12 gpurun_out/pytest_gpu_full.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_c3.json
UPY_LIB=$PWD/paper_2403_13839_b200/_variants/allocnoinl.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_var_allocnoinl.json
timeout 600 python bench.py --workload c3_311 --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_c3_311.json
timeout 300 python bench.py --workload c2_311 --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_c2_311.json
ls -la gpurun_out
