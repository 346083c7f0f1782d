# C4 slot-count sweep (arena budget experiment).  Outputs in gpurun_out/.
mkdir -p gpurun_out
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=memory.total,memory.used --format=csv | tee gpurun_out/mem.txt
for s in 12288 24576 49152 65536; do
  timeout 600 python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu --pyc 0 --slots $s --arena-bytes 2621440 2>&1 | tail -1 | tee gpurun_out/c4_slots_$s.json
done
