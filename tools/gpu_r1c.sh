# decode kernel v2 (TMA bulk pipeline): parity, C3/C2 benches, ncu of the decode kernel
set -x
mkdir -p gpurun_out /tmp/ncu
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 | tee gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench_c3.json
timeout 300 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench_c2.json
timeout 600 python bench.py --workload c2x --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench_c2x.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --pyc 0 > gpurun_out/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:upy_decode -s 2 -c 1 -o /tmp/ncu/decode -f python bench.py --no-cpu --steps 1 --warmup 3 --pyc 0 > gpurun_out/ncu_decode.log 2>&1
ncu -i /tmp/ncu/decode.ncu-rep --page raw --csv > gpurun_out/ncu_decode_raw.csv 2>&1
ncu -i /tmp/ncu/decode.ncu-rep --page details --csv > gpurun_out/ncu_decode_details.csv 2>&1
ncu -i /tmp/ncu/decode.ncu-rep --page source --csv > /tmp/ncu/decode_source.csv 2>&1; gzip -c /tmp/ncu/decode_source.csv > gpurun_out/ncu_decode_source.csv.gz
cp /tmp/ncu/decode.ncu-rep gpurun_out/
ls -la gpurun_out
