# code-size fix (no unrolled zero/copy loops), decode v3, schedule removal: tests with durations, benches, variants
set -x
mkdir -p gpurun_out /tmp/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1800 python -m pytest tests -m gpu -q --durations=25 -p no:cacheprovider > gpurun_out/pytest_gpu_full.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
tail -40 gpurun_out/pytest_gpu_full.txt
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_c3.json
UPY_LIB=$PWD/paper_2403_13839_b200/_variants/dec5.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_var_dec5.json
UPY_LIB=$PWD/paper_2403_13839_b200/_variants/dclocal2.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_var_dclocal2.json
timeout 600 python bench.py --workload c2x --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c2x.json
timeout 300 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --pyc 0 > gpurun_out/ncu_launches.log 2>&1
ls -la gpurun_out
