# C4 decode iteration: GPU tests, C4 (3.10) line (no extras), decode launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pt.txt
timeout 900 python bench.py --workload c4 --no-extra --pyc 0 --no-cpu --steps 1 --warmup 1 2>&1 | tail -1 > gpurun_out/bc4.json
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:decode -c 4 --csv --log-file gpurun_out/l_c4.csv python bench.py --workload c4 --no-extra --pyc 0 --no-cpu --steps 1 --warmup 1 > gpurun_out/ncu_c4.log 2>&1
