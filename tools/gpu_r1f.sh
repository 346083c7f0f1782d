# out-of-line slow paths + Dc on the stack + decode minb5 + KeyError message fix
set -x
mkdir -p gpurun_out /tmp/ncu
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q --durations=10 -p no:cacheprovider > gpurun_out/pytest_gpu_full.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
tail -15 gpurun_out/pytest_gpu_full.txt
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_c3.json
if [ -f paper_2403_13839_b200/_variants/inl.so ]; then
UPY_LIB=$PWD/paper_2403_13839_b200/_variants/inl.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --pyc 0 2>&1 | tail -1 > gpurun_out/bench_var_inl.json
fi
timeout 600 python bench.py --workload c2x --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c2x.json
timeout 600 python bench.py --workload c3_311 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c3_311.json
timeout 900 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c4.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --pyc 0 > gpurun_out/ncu_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:upy_decompile -c 1 -o /tmp/ncu/decompile -f python bench.py --no-cpu --steps 1 --warmup 1 --pyc 0 --objects 262144 > gpurun_out/ncu_decompile.log 2>&1
ncu -i /tmp/ncu/decompile.ncu-rep --page raw --csv > gpurun_out/ncu_decompile_raw.csv 2>&1
ncu -i /tmp/ncu/decompile.ncu-rep --page details --csv > gpurun_out/ncu_decompile_details.csv 2>&1
ncu -i /tmp/ncu/decompile.ncu-rep --page source --csv > /tmp/ncu/decompile_source.csv 2>&1; gzip -c /tmp/ncu/decompile_source.csv > gpurun_out/ncu_decompile_source.csv.gz
timeout 600 ncu --set full --clock-control none --import-source on -k regex:upy_decode -s 2 -c 1 -o /tmp/ncu/decode -f python bench.py --no-cpu --steps 1 --warmup 3 --pyc 0 > gpurun_out/ncu_decode.log 2>&1
ncu -i /tmp/ncu/decode.ncu-rep --page raw --csv > gpurun_out/ncu_decode_raw.csv 2>&1
ls -la gpurun_out
