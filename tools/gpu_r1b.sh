# Re-entry check: parity tests + smoke + bench (both decompile schedules)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench_c3_s0.json
timeout 600 python bench.py --steps 5 --warmup 3 --schedule 1 --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench_c3_s1.json
timeout 600 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench_c4_s0.json
timeout 600 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu --schedule 1 2>&1 | tail -1 | tee gpurun_out/bench_c4_s1.json
