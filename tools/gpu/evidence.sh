# Evidence run: smoke, GPU tests, the new default bench line (distinct C3 corpus
# + extras), the reference arm, an ncu DRAM-traffic launch list and a full-set
# capture of the decompile kernel.  Outputs in gpurun_out/.
mkdir -p gpurun_out /tmp/ncu
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.txt
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 | tee gpurun_out/pytest_gpu.txt
timeout 1200 python bench.py 2>&1 | tail -1 | tee gpurun_out/bench.json
timeout 600 python bench.py --impl reference 2>&1 | tail -1 | tee gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/traffic_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu --pyc 0 --no-extra \
  > gpurun_out/ncu_traffic.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:upy_decompile -s 1 -c 1 \
  -o /tmp/ncu/decompile -f python bench.py --no-cpu --pyc 0 --no-extra --steps 1 --warmup 2 --objects 262144 \
  > gpurun_out/ncu_decompile.log 2>&1
ncu -i /tmp/ncu/decompile.ncu-rep --page raw --csv > gpurun_out/ncu_decompile_raw.csv 2>&1
ncu -i /tmp/ncu/decompile.ncu-rep --page source --csv > /tmp/ncu/decompile_source.csv 2>&1
gzip -c /tmp/ncu/decompile_source.csv > gpurun_out/ncu_decompile_source.csv.gz
ls -la gpurun_out
