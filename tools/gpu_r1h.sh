# source-level profile of the current decompile kernel; occupancy (slot count) sweep at fixed code
set -x
mkdir -p gpurun_out /tmp/ncu
for s in 75776 113664; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 --slots $s 2>&1 | tail -1 > gpurun_out/bench_slots_$s.json
done
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:upy_decompile -c 1 -o /tmp/ncu/decompile -f python bench.py --no-cpu --steps 1 --warmup 1 --pyc 0 --objects 262144 > gpurun_out/ncu_decompile.log 2>&1
ncu -i /tmp/ncu/decompile.ncu-rep --page raw --csv > gpurun_out/ncu_decompile_raw.csv 2>&1
ncu -i /tmp/ncu/decompile.ncu-rep --page details --csv > gpurun_out/ncu_decompile_details.csv 2>&1
ncu -i /tmp/ncu/decompile.ncu-rep --page source --csv > /tmp/ncu/decompile_source.csv 2>&1; gzip -c /tmp/ncu/decompile_source.csv > gpurun_out/ncu_decompile_source.csv.gz
timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_c5.json
ls -la gpurun_out
