mkdir -p gpurun_out
for lib in libupy_cO1pO1.so libupy_cO3pO1.so libupy_cO3pO3.so; do
  echo "== $lib"
  UPY_LIB=paper_2403_13839_b200/$lib timeout 600 python bench.py --no-cpu --steps 3 --warmup 2 2>&1 | tail -1 > gpurun_out/exp_$lib.json
  python tools/show_bench.py gpurun_out/exp_$lib.json
done
