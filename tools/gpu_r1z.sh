# per-thread arena slot size sweep (C3): default (64 KB + 160 B x max code len) vs smaller slots
set -x
mkdir -p gpurun_out
rm -f gpurun_out/bench_*.json
for r in 1 2; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_default_$r.json
  for ab in 65536 40960; do
    timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 --arena-bytes $ab 2>&1 | tail -1 > gpurun_out/bench_ab${ab}_$r.json
  done
done
ls -la gpurun_out
