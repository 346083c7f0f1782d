# Round-end evidence on the committed tree (after the 3.11 lane decode kernel): smoke, GPU tier,
# default bench line (with extras), reference arm, torchrun N=1 lines, the default line's
# launch list with DRAM bytes, and a full capture of the 3.11 lane decode kernel.
mkdir -p gpurun_out /tmp/ncu
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee gpurun_out/final_smoke.txt
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 | tee gpurun_out/final_pytest.txt
timeout 1200 python bench.py 2>&1 | tail -1 > gpurun_out/final_bench.json
timeout 900 python bench.py --impl reference 2>&1 | tail -1 > gpurun_out/final_bench_ref.json
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 \
  bench.py --gpus 1 --no-extra 2>&1 | tail -1 > gpurun_out/final_bench_torchrun1.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 \
  bench.py --impl reference --gpus 1 2>&1 | tail -1 > gpurun_out/final_bench_ref_torchrun.json
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu --pyc 0 --no-extra \
  > gpurun_out/ncu_launches_final.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lane -s 1 -c 1 -o /tmp/ncu/lane311 -f \
  python bench.py --workload c3_311 --no-extra --pyc 0 --no-cpu --steps 1 --warmup 3 > gpurun_out/ncu_lane311.log 2>&1
ncu -i /tmp/ncu/lane311.ncu-rep --page raw --csv > gpurun_out/ncu_lane311_raw.csv 2>&1
ncu -i /tmp/ncu/lane311.ncu-rep --page source --csv --print-source sass > /tmp/ncu/lane311_src.csv 2>&1
gzip -c /tmp/ncu/lane311_src.csv > gpurun_out/ncu_lane311_source.csv.gz
ls -la gpurun_out
