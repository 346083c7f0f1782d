python -m paper_2403_13839_b200.build >/dev/null
for lib in libupy_cuda.so libupy_minb4.so libupy_minb8.so; do
  for ab in 0 196608; do
    echo "== $lib arena_bytes=$ab"
    UPY_LIB=paper_2403_13839_b200/$lib timeout 600 python bench.py --no-cpu --steps 3 --warmup 2 --arena-bytes $ab 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), d['kernel_ms'], d['parity']['mismatches'])"
  done
done
