# text helpers inline + loop invariants hoisted + small-batch latency mode
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_full.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
tail -3 gpurun_out/pytest_gpu_full.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for r in 1 2; do timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_c3_$r.json; done
timeout 300 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c2.json
timeout 300 python bench.py --workload c2_311 --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c2_311.json
ls -la gpurun_out
