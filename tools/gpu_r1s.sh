# A/B: section bases in the context (main) vs + per-instruction helpers inlined (syminl variant)
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_full.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
tail -3 gpurun_out/pytest_gpu_full.txt
for r in 1 2; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_main_$r.json
  if [ -f paper_2403_13839_b200/_variants/syminl.so ]; then
  UPY_LIB=$PWD/paper_2403_13839_b200/_variants/syminl.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_syminl_$r.json
  fi
done
ls -la gpurun_out
