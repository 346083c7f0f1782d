# 3.11 decode iteration: GPU tests, C3-3.11 and C3 bench lines (no extras), launch list of the decode kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pt.txt
timeout 600 python bench.py --workload c3_311 --no-extra --pyc 0 --no-cpu --steps 3 2>&1 | tail -1 > gpurun_out/b311.json
timeout 600 python bench.py --no-extra --pyc 0 --no-cpu --steps 3 2>&1 | tail -1 > gpurun_out/b310.json
for w in c3_311 c3; do
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:decode -c 4 --csv --log-file gpurun_out/l_$w.csv python bench.py --workload $w --no-extra --pyc 0 --no-cpu --steps 1 --warmup 3 > gpurun_out/ncu_$w.log 2>&1
done
