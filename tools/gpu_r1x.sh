# A/B: compile-time-sized clears for anew<T> (anewconst) vs mkconst
set -x
mkdir -p gpurun_out
rm -f gpurun_out/bench_*.json
for r in 1 2; do
  UPY_LIB=$PWD/paper_2403_13839_b200/_variants/mkconst.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_mkconst_$r.json
  UPY_LIB=$PWD/paper_2403_13839_b200/_variants/anewconst.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_anewconst_$r.json
done
UPY_LIB=$PWD/paper_2403_13839_b200/_variants/anewconst.so timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_anewconst.txt 2>&1; tail -2 gpurun_out/pytest_anewconst.txt
ls -la gpurun_out
