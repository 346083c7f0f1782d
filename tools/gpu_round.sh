# One GPU session: parity tests, benches, ncu evidence.  Outputs in gpurun_out/
# (kept < 64 MiB: full ncu reports stay in /tmp on the box, CSV exports come back).
set -x
mkdir -p gpurun_out /tmp/ncu
python -m paper_2403_13839_b200.build
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench_c3.json
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench_c4.json
timeout 900 python bench.py --workload c3_311 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench_c3_311.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench_ref.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench_torchrun1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:upy_decode -s 2 -c 1 -o /tmp/ncu/decode -f python bench.py --no-cpu --steps 1 --warmup 3 > gpurun_out/ncu_decode.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:upy_decompile -s 1 -c 1 -o /tmp/ncu/decompile -f python bench.py --no-cpu --steps 1 --warmup 2 --objects 262144 > gpurun_out/ncu_decompile.log 2>&1
for k in decode decompile; do
  ncu -i /tmp/ncu/$k.ncu-rep --page raw --csv > gpurun_out/ncu_${k}_raw.csv 2>&1
  ncu -i /tmp/ncu/$k.ncu-rep --page details --csv > gpurun_out/ncu_${k}_details.csv 2>&1
  ncu -i /tmp/ncu/$k.ncu-rep --page source --csv > /tmp/ncu/${k}_source.csv 2>&1
  gzip -c /tmp/ncu/${k}_source.csv > gpurun_out/ncu_${k}_source.csv.gz
  sz=$(stat -c %s /tmp/ncu/$k.ncu-rep)
  if [ "$sz" -lt 25000000 ]; then cp /tmp/ncu/$k.ncu-rep gpurun_out/; fi
done
ls -la gpurun_out
