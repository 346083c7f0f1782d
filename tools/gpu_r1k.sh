# round-1 evidence run on the committed tree: tests, all workloads, reference arm, torchrun, ncu evidence
set -x
mkdir -p gpurun_out /tmp/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.txt
timeout 1200 python -m pytest tests -m gpu -q --durations=5 -p no:cacheprovider > gpurun_out/pytest_gpu_full.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
tail -4 gpurun_out/pytest_gpu_full.txt
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_c3.json
timeout 600 python bench.py --impl reference 2>&1 | tail -1 > gpurun_out/bench_ref.json
timeout 300 python bench.py --workload c2 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c2.json
timeout 600 python bench.py --workload c2x --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c2x.json
timeout 600 python bench.py --workload c3_311 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c3_311.json
timeout 900 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c4.json
timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_c5.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_torchrun1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu --pyc 0 > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu --pyc 0 > gpurun_out/ncu_traffic.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_c3_311.csv python bench.py --workload c3_311 --steps 1 --warmup 3 --no-cpu --pyc 0 > gpurun_out/ncu_traffic311.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:upy_decode -s 2 -c 1 -o /tmp/ncu/decode -f python bench.py --no-cpu --steps 1 --warmup 3 --pyc 0 > gpurun_out/ncu_decode.log 2>&1
ncu -i /tmp/ncu/decode.ncu-rep --page raw --csv > gpurun_out/ncu_decode_raw.csv 2>&1
ncu -i /tmp/ncu/decode.ncu-rep --page details --csv > gpurun_out/ncu_decode_details.csv 2>&1
ls -la gpurun_out
timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu --pyc 0 > gpurun_out/bench_c5.log 2>&1; tail -1 gpurun_out/bench_c5.log > gpurun_out/bench_c5.json
