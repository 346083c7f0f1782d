set -x
python -m paper_2403_13839_b200.build
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --no-cpu --steps 2 --warmup 1 --objects 200000 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:upy_decode -c 1 -o gpurun_out/prof_decode_r01 -f python bench.py --no-cpu --steps 1 --warmup 1 --objects 1000000 > gpurun_out/ncu_decode.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:upy_decompile -c 1 -o gpurun_out/prof_decompile_r01 -f python bench.py --no-cpu --steps 1 --warmup 1 --objects 65536 > gpurun_out/ncu_decompile.log 2>&1
ls -la gpurun_out
