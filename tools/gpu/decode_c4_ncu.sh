# full ncu capture of the main decode kernel on C4 (one launch)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:upy_decode_kernel -s 1 -c 1 -o gpurun_out/dec_c4 -f \
  python bench.py --workload c4 --no-extra --pyc 0 --no-cpu --steps 1 --warmup 1 > gpurun_out/ncu_c4f.log 2>&1
