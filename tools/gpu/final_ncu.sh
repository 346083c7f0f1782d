mkdir -p gpurun_out /tmp/ncu
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu --pyc 0 --no-extra \
  > gpurun_out/ncu_launches_final.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:upy_decompile -s 1 -c 1 \
  -o /tmp/ncu/decompile -f python bench.py --no-cpu --pyc 0 --no-extra --steps 1 --warmup 2 --objects 262144 \
  > gpurun_out/ncu_decompile_final.log 2>&1
ncu -i /tmp/ncu/decompile.ncu-rep --page raw --csv > gpurun_out/ncu_decompile_final_raw.csv 2>&1
