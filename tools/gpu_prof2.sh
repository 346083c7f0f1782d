python -m paper_2403_13839_b200.build >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --no-cpu --steps 5 --warmup 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), d['kernel_ms'], d['parity'], d['e2e']['value'])"
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:upy_decompile -c 1 -o gpurun_out/prof_decompile_r01b -f python bench.py --no-cpu --steps 1 --warmup 1 --objects 262144 > gpurun_out/ncu_decompile_b.log 2>&1
