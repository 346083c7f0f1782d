set -x
python -m paper_2403_13839_b200.build
timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 --objects 100000 2>&1 | tail -5
timeout 900 python bench.py --no-cpu --steps 3 --warmup 3 2>&1 | tail -5
