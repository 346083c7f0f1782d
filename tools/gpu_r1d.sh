# GPU test durations + decompile-kernel register-cap variants + ncu source profile of the decompile kernel
set -x
mkdir -p gpurun_out /tmp/ncu
timeout 2400 python -m pytest tests -m gpu -q --durations=0 -p no:cacheprovider > gpurun_out/pytest_gpu_full.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
tail -5 gpurun_out/pytest_gpu_full.txt
for v in minb4 minb5 minb6 minb10; do
  if [ -f paper_2403_13839_b200/_variants/$v.so ]; then
    UPY_LIB=$PWD/paper_2403_13839_b200/_variants/$v.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_var_$v.json
  fi
done
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:upy_decompile -c 1 -o /tmp/ncu/decompile -f python bench.py --no-cpu --steps 1 --warmup 1 --pyc 0 --objects 262144 > gpurun_out/ncu_decompile.log 2>&1
ncu -i /tmp/ncu/decompile.ncu-rep --page raw --csv > gpurun_out/ncu_decompile_raw.csv 2>&1
ncu -i /tmp/ncu/decompile.ncu-rep --page details --csv > gpurun_out/ncu_decompile_details.csv 2>&1
ncu -i /tmp/ncu/decompile.ncu-rep --page source --csv > /tmp/ncu/decompile_source.csv 2>&1; gzip -c /tmp/ncu/decompile_source.csv > gpurun_out/ncu_decompile_source.csv.gz
ls -la gpurun_out
