# A/B: node construction with constant sizes + straight-line clears (mkconst) vs main
set -x
mkdir -p gpurun_out
rm -f gpurun_out/bench_*.json
for r in 1 2; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_main_$r.json
  UPY_LIB=$PWD/paper_2403_13839_b200/_variants/mkconst.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_mkconst_$r.json
done
UPY_LIB=$PWD/paper_2403_13839_b200/_variants/mkconst.so timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_mkconst.txt 2>&1; tail -2 gpurun_out/pytest_mkconst.txt
ls -la gpurun_out
