# A/B in one session: text helpers out of line (main) vs inline (variant), 3 runs each interleaved
set -x
mkdir -p gpurun_out
for r in 1 2 3; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_main_$r.json
  UPY_LIB=$PWD/paper_2403_13839_b200/_variants/textinl.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_textinl_$r.json
done
ls -la gpurun_out
