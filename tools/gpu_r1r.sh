set -x
mkdir -p gpurun_out /tmp/ncu
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:upy_decompile -c 1 -o /tmp/ncu/decompile -f python bench.py --no-cpu --steps 1 --warmup 1 --pyc 0 --objects 262144 > gpurun_out/ncu_decompile.log 2>&1
ncu -i /tmp/ncu/decompile.ncu-rep --page raw --csv > gpurun_out/ncu_decompile_raw.csv 2>&1
ncu -i /tmp/ncu/decompile.ncu-rep --page source --csv > /tmp/ncu/decompile_source.csv 2>&1; gzip -c /tmp/ncu/decompile_source.csv > gpurun_out/ncu_decompile_source.csv.gz
ls -la gpurun_out
