# full ncu capture of the 3.11 lane decode kernel (C3-3.11, one launch)
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lane -s 1 -c 1 -o gpurun_out/lane311 -f \
  python bench.py --workload c3_311 --no-extra --pyc 0 --no-cpu --steps 1 --warmup 3 > gpurun_out/ncu2.log 2>&1
