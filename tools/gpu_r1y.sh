# A/B/C: text helpers t_putn/t_puts out of line (textool), + t_put (alltextool) vs main
set -x
mkdir -p gpurun_out
rm -f gpurun_out/bench_*.json
for r in 1 2; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_main_$r.json
  for v in textool alltextool; do
    UPY_LIB=$PWD/paper_2403_13839_b200/_variants/$v.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_${v}_$r.json
  done
done
ls -la gpurun_out
