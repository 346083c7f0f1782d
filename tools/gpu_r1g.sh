# optab in shared memory, 3.11 decode from shared memory, KeyError message; stagger variant
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q --durations=5 -p no:cacheprovider > gpurun_out/pytest_gpu_full.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
tail -6 gpurun_out/pytest_gpu_full.txt
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_c3.json
if [ -f paper_2403_13839_b200/_variants/stagger.so ]; then
UPY_LIB=$PWD/paper_2403_13839_b200/_variants/stagger.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_var_stagger.json
fi
timeout 600 python bench.py --workload c3_311 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c3_311.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_ref.json
ls -la gpurun_out
