set -x
mkdir -p gpurun_out
python -m paper_2403_13839_b200.build
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS} 2>&1 | tail -1 | tee gpurun_out/bench_last.json
