# Timing experiment: the decompile kernel without the emit stage (output is wrong by
# construction; only the kernel time matters) vs the full kernel, same session.
mkdir -p gpurun_out
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for v in base noemit base noemit; do
  if [ $v = base ]; then L=; else L=paper_2403_13839_b200/_variants/$v.so; fi
  UPY_LIB=$L timeout 900 python bench.py --no-cpu --pyc 0 --no-extra --steps 3 2>&1 | tail -1 > gpurun_out/bench_e_$v.json
  python -c "import json; d=json.load(open('gpurun_out/bench_e_$v.json')); print('$v', d['kernel_ms'])" | tee -a gpurun_out/ab_e.txt
done
ncu --metrics sm__icc_request_hit_rate.pct,gcc__cache_requests_type_instruction.sum,gcc__cache_requests_type_instruction.sum.pct_of_peak_sustained_elapsed,smsp__average_warp_latency_per_inst_issued.ratio,gpu__time_duration.sum \
  -k regex:upy_decompile -s 1 -c 1 --csv python bench.py --no-cpu --pyc 0 --no-extra --steps 1 --warmup 1 --objects 262144 > gpurun_out/icc_base.csv 2>&1
UPY_LIB=paper_2403_13839_b200/_variants/noemit.so ncu --metrics sm__icc_request_hit_rate.pct,gcc__cache_requests_type_instruction.sum,gcc__cache_requests_type_instruction.sum.pct_of_peak_sustained_elapsed,smsp__average_warp_latency_per_inst_issued.ratio,gpu__time_duration.sum \
  -k regex:upy_decompile -s 1 -c 1 --csv python bench.py --no-cpu --pyc 0 --no-extra --steps 1 --warmup 1 --objects 262144 > gpurun_out/icc_noemit.csv 2>&1
