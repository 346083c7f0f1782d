# A/B: cicc -O2 vs -O3 for the decompile kernel (instruction-cache pressure is back at 33 stall cycles/issue)
set -x
mkdir -p gpurun_out
rm -f gpurun_out/bench_*.json
for r in 1 2; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_main_$r.json
  UPY_LIB=$PWD/paper_2403_13839_b200/_variants/cicco2.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_cicco2_$r.json
done
ls -la gpurun_out
