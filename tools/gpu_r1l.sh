# Ins copy without zeroing, pinned fetch + pyc breakdown; ptxas -O2 / -O3 variants of the decompile kernel
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_full.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
tail -3 gpurun_out/pytest_gpu_full.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c3.json
for v in ptxo2 ptxo3; do
  if [ -f paper_2403_13839_b200/_variants/$v.so ]; then
    UPY_LIB=$PWD/paper_2403_13839_b200/_variants/$v.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_var_$v.json
  fi
done
ls -la gpurun_out
