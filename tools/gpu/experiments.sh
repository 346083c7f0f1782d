# Round-2 GPU experiments, one function each (outputs in gpurun_out/):
#   bash tools/gpu/experiments.sh <name> [...]
# c4_slots   C4 throughput vs concurrent arena slots (profiles/r02/bench_c4_slots_*.json)
# stages     thread-cycles per pipeline stage (needs tools/build_variant.sh prof -DUPY_PHASE_PROF)
# noemit     decompile kernel without the emit stage vs full, + icache metrics (variant noemit -DUPY_SKIP_EMIT)
# variant    same-session A/B of a variant library: VARIANT=<name> (built by tools/build_variant.sh)
# stackscan  stack-scan kernel: timing on C3 / C4 and a full ncu capture
# decode311  3.11 decode timing and a full ncu capture on C3-3.11
# schedule   root order input vs largest-tree-first (api.root_cost_order) on C2x / C4 / C2
# sync       warp-synchronous root fetch (upy_options.schedule = 1) x root order
# split      schedule 3 (separate tree and emit kernels) vs the fused kernel, parity forced on
# c5         the 16M-object corpus on one GPU, and torchrun N=1 lines (ours and the reference arm)
set -u
mkdir -p gpurun_out /tmp/ncu
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
V=paper_2403_13839_b200/_variants
c4_slots() {
  for s in 12288 24576 49152; do
    timeout 600 python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu --pyc 0 --slots $s --arena-bytes 2621440 \
      2>&1 | tail -1 > gpurun_out/c4_slots_$s.json
  done
}
stages() {
  UPY_LIB=$V/prof.so timeout 600 python tools/stage_prof.py c3_310 c3_311 | tee gpurun_out/stage_prof_c3.txt
  UPY_LIB=$V/prof.so timeout 900 python tools/stage_prof.py c4_310 c4_311 --objects 16384 | tee gpurun_out/stage_prof_c4.txt
}
ab() {  # ab <variant> : base / variant / base / variant, kernel times
  for v in base $1 base $1; do
    if [ $v = base ]; then L=; else L=$V/$v.so; fi
    UPY_LIB=$L timeout 900 python bench.py --no-cpu --pyc 0 --no-extra --steps 3 2>&1 | tail -1 > gpurun_out/ab_$v.json
    python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', d['kernel_ms'], d['parity'])" \
      | tee -a gpurun_out/ab_$1.txt
  done
}
icc() {  # icc <lib or empty> <tag>
  M=sm__icc_request_hit_rate.pct,gcc__cache_requests_type_instruction.sum,gcc__cache_requests_type_instruction.sum.pct_of_peak_sustained_elapsed,smsp__average_warp_latency_per_inst_issued.ratio,gpu__time_duration.sum
  UPY_LIB=$1 ncu --metrics $M -k regex:upy_decompile -s 1 -c 1 --csv \
    python bench.py --no-cpu --pyc 0 --no-extra --steps 1 --warmup 1 --objects 262144 > gpurun_out/icc_$2.csv 2>&1
}
noemit() { ab noemit; icc "" base; icc $V/noemit.so noemit; }
variant() { ab "$VARIANT"; }
stackscan() {
  timeout 900 python bench.py --no-cpu --pyc 0 --no-extra 2>&1 | tail -1 > gpurun_out/bench_stackscan_c3.json
  timeout 900 python bench.py --workload c4 --no-cpu --pyc 0 --steps 1 --warmup 1 2>&1 | tail -1 > gpurun_out/bench_stackscan_c4.json
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:upy_stackscan -s 1 -c 1 -o /tmp/ncu/stackscan -f \
    python bench.py --no-cpu --pyc 0 --no-extra --steps 1 --warmup 1 > gpurun_out/ncu_stackscan.log 2>&1
  ncu -i /tmp/ncu/stackscan.ncu-rep --page raw --csv > gpurun_out/ncu_stackscan_raw.csv 2>&1
}
decode311() {
  timeout 900 python bench.py --workload c3_311 --no-cpu --pyc 0 --no-extra --steps 3 2>&1 | tail -1 > gpurun_out/bench_decode311.json
  timeout 600 ncu --set full --clock-control none -k regex:upy_decode -s 3 -c 1 --csv --page raw \
    python bench.py --workload c3_311 --no-cpu --pyc 0 --no-extra --steps 1 --warmup 2 > gpurun_out/ncu_decode311_raw.csv 2>&1
}
schedule() {  # root order: input vs largest-tree-first, on the mixed-size shapes
  for wl in c2x c4 c2; do
    for sc in input cost input cost; do
      timeout 900 python bench.py --workload $wl --schedule $sc --no-cpu --pyc 0 --no-extra --steps 2 --warmup 1 \
        2>&1 | tail -1 > gpurun_out/sched_${wl}_$sc.json
      python -c "import json; d=json.load(open('gpurun_out/sched_${wl}_$sc.json')); print('$wl $sc', round(d['value']), d['kernel_ms'], d['parity'])" \
        | tee -a gpurun_out/schedule.txt
    done
  done
}
sync() {  # warp-synchronous root fetch x root order, distinct C3 and the tiled C4
  for wl in c3 c4; do
    for sc in cost cost+sync similar similar+sync input+sync; do
      st=2; [ $wl = c4 ] && st=1
      timeout 900 python bench.py --workload $wl --schedule $sc --no-cpu --pyc 0 --no-extra --steps $st --warmup 1 \
        2>&1 | tail -1 > gpurun_out/sync_${wl}_$sc.json
      python -c "import json; d=json.load(open('gpurun_out/sync_${wl}_$sc.json')); print('$wl $sc', round(d['value']), d['kernel_ms'], d['parity'])" \
        | tee -a gpurun_out/sync.txt
    done
  done
}
quick_ss() {  # stack-scan parity + timing on C3 / C4
  timeout 900 python -m pytest -m gpu -x -q tests/test_stackscan.py 2>&1 | tail -3 | tee gpurun_out/pytest_ss.txt
  stackscan
  python -c "import json; [print(f, json.load(open('gpurun_out/'+f+'.json'))['roofline_stackscan']) for f in ('bench_stackscan_c3','bench_stackscan_c4')]" | tee gpurun_out/ss.txt
}
shape() {  # opcode-prefix order (args ignored), with and without warp-synchronous fetch, on distinct C3
  for sc in cost shape shape+sync cost shape+sync; do
    timeout 900 python bench.py --workload c3 --schedule $sc --no-cpu --pyc 0 --no-extra --steps 3 --warmup 2 \
      2>&1 | tail -1 > gpurun_out/shape_c3_$sc.json
    python -c "import json; d=json.load(open('gpurun_out/shape_c3_$sc.json')); print('c3 $sc', round(d['value']), d['kernel_ms'], d['parity'])" \
      | tee -a gpurun_out/shape.txt
  done
}
coemit() {  # statement-parallel emission: parity on every golden set (throughput mode) + A/B on C3 / C3-3.11 / C4
  UPY_SCHEDULE=cost+coemit timeout 1500 python -m pytest -m gpu -x -q tests/test_golden_gpu.py tests/test_cli.py \
    2>&1 | tail -4 | tee gpurun_out/pytest_coemit.txt
  for wl in c3 c3_311; do
    for sc in cost cost+coemit cost cost+coemit; do
      timeout 900 python bench.py --workload $wl --schedule $sc --no-cpu --pyc 0 --no-extra --steps 3 --warmup 2 \
        2>&1 | tail -1 > gpurun_out/coemit_${wl}_$sc.json
      python -c "import json; d=json.load(open('gpurun_out/coemit_${wl}_$sc.json')); print('$wl $sc', round(d['value']), d['kernel_ms'], d['parity'])" \
        | tee -a gpurun_out/coemit.txt
    done
  done
  for sc in input input+coemit; do
    timeout 900 python bench.py --workload c4 --schedule $sc --no-cpu --pyc 0 --no-extra --steps 1 --warmup 1 \
      2>&1 | tail -1 > gpurun_out/coemit_c4_$sc.json
    python -c "import json; d=json.load(open('gpurun_out/coemit_c4_$sc.json')); print('c4 $sc', round(d['value']), d['kernel_ms'], d['parity'])" \
      | tee -a gpurun_out/coemit.txt
  done
}
dshape() {  # device-side opcode-shape orders (1, 2, 4 chained 64-bit sorts) vs cost, distinct C3
  for sc in cost dshape1 dshape2 dshape4 cost dshape2 dshape4; do
    timeout 900 python bench.py --workload c3 --schedule $sc --no-cpu --pyc 0 --no-extra --steps 3 --warmup 2 \
      2>&1 | tail -1 > gpurun_out/dshape_c3_$sc.json
    python -c "import json; d=json.load(open('gpurun_out/dshape_c3_$sc.json')); print('c3 $sc', round(d['value']), round(d['e2e']['value']), d['kernel_ms'], d['parity'])" \
      | tee -a gpurun_out/dshape.txt
  done
}
coemit2() {  # coemit v2 (parallel headers, one scratch per round): parity forced on + C3 / C4 timing
  UPY_SCHEDULE=cost+coemit timeout 1500 python -m pytest -m gpu -x -q tests/test_golden_gpu.py tests/test_cli.py \
    2>&1 | tail -3 | tee gpurun_out/pytest_coemit2.txt
  for sc in cost cost+coemit cost cost+coemit; do
    timeout 900 python bench.py --workload c3 --schedule $sc --no-cpu --pyc 0 --no-extra --steps 3 --warmup 2 \
      2>&1 | tail -1 > gpurun_out/coemit2_c3_$sc.json
    python -c "import json; d=json.load(open('gpurun_out/coemit2_c3_$sc.json')); print('c3 $sc', round(d['value']), d['kernel_ms'], d['parity'])" \
      | tee -a gpurun_out/coemit2.txt
  done
  for sc in input+thread input+coemit; do
    timeout 900 python bench.py --workload c4 --schedule $sc --no-cpu --pyc 0 --no-extra --steps 1 --warmup 1 \
      2>&1 | tail -1 > gpurun_out/coemit2_c4_$sc.json
    python -c "import json; d=json.load(open('gpurun_out/coemit2_c4_$sc.json')); print('c4 $sc', round(d['value']), d['kernel_ms'], d['parity'])" \
      | tee -a gpurun_out/coemit2.txt
  done
}
coemit_split() {  # where coemit's time goes on C3: tree + warp sync only (variant nocoemit) vs full
  for v in base nocoemit base nocoemit; do
    if [ $v = base ]; then L=; else L=$V/$v.so; fi
    UPY_LIB=$L timeout 900 python bench.py --workload c3 --schedule cost+coemit --no-cpu --pyc 0 --no-extra --steps 3 \
      2>&1 | tail -1 > gpurun_out/cs_$v.json
    python -c "import json; d=json.load(open('gpurun_out/cs_$v.json')); print('$v', d['kernel_ms'])" | tee -a gpurun_out/coemit_split.txt
  done
}
split() {  # schedule 3 (tree kernel + emit kernel): parity forced on + C3 / C3-3.11 timing + icache
  : UPY_SCHEDULE=cost+split timeout 1500 python -m pytest -m gpu -x -q tests/test_golden_gpu.py tests/test_cli.py \
    2>&1 | tail -3 | tee gpurun_out/pytest_split.txt
  for wl in c3 c3_311; do
    for sc in cost cost+split cost cost+split; do
      timeout 900 python bench.py --workload $wl --schedule $sc --no-cpu --pyc 0 --no-extra --steps 3 --warmup 2 \
        2>&1 | tail -1 > gpurun_out/split_${wl}_$sc.json
      python -c "import json; d=json.load(open('gpurun_out/split_${wl}_$sc.json')); print('$wl $sc', round(d['value']), d['kernel_ms'], d['parity'])" \
        | tee -a gpurun_out/split.txt
    done
  done
  M=sm__icc_request_hit_rate.pct,gcc__cache_requests_type_instruction.sum.pct_of_peak_sustained_elapsed,smsp__average_warp_latency_per_inst_issued.ratio,smsp__thread_inst_executed_per_inst_executed.ratio,dram__bytes.sum,gpu__time_duration.sum
  ncu --metrics $M -k regex:"upy_(tree|emit|decompile)" -c 3 --csv \
    python bench.py --schedule cost+split --no-cpu --pyc 0 --no-extra --steps 1 --warmup 1 --objects 262144 > gpurun_out/icc_split.csv 2>&1
}
split2() {  # split as the API default for short objects: full GPU tests, default line, C5, C2x
  timeout 1800 python -m pytest -m gpu -x -q tests 2>&1 | tail -3 | tee gpurun_out/pytest_split2.txt
  timeout 1200 python bench.py 2>&1 | tail -1 > gpurun_out/bench_split2.json
  timeout 1800 python bench.py --workload c5 --no-cpu --pyc 0 --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_c5_split2.json
  for sc in auto input+thread; do
    timeout 900 python bench.py --workload c2x --schedule $sc --no-cpu --pyc 0 --no-extra --steps 3 --warmup 2 \
      2>&1 | tail -1 > gpurun_out/split2_c2x_$sc.json
  done
  for f in gpurun_out/bench_split2.json gpurun_out/bench_c5_split2.json gpurun_out/split2_c2x_*.json; do
    python -c "import json,sys; d=json.load(open('$f')); print('$f', d['config']['schedule'], round(d['value']), round(d['e2e']['value']), d['kernel_ms'], d['parity'], d['gpu_launches'])" \
      | tee -a gpurun_out/split2.txt
  done
}
split_minb() {  # split kernels' launch bounds: variants em6/em12 (emit) tr6/tr10 (tree) vs base, C3 + C2x
  for round in 1 2; do
    for v in base em6 em12 tr6 tr10; do
      if [ $v = base ]; then L=; else L=$V/$v.so; fi
      for wl in c3 c2x; do
        UPY_LIB=$L timeout 900 python bench.py --workload $wl --schedule auto --no-cpu --pyc 0 --no-extra --steps 3 --warmup 2 \
          2>&1 | tail -1 > gpurun_out/minb_${wl}_$v.json
        python -c "import json; d=json.load(open('gpurun_out/minb_${wl}_$v.json')); print('$wl $v', d['config']['schedule'], round(d['value']), d['kernel_ms'], d['parity']['mismatches'])" \
          | tee -a gpurun_out/split_minb.txt
      done
    done
  done
}
split_big() {  # split on many chunks (C5 16M) and on long objects (C4, explicit 2.5 MB slots)
  for sc in cost+split cost+thread; do
    timeout 1800 python bench.py --workload c5 --schedule $sc --no-cpu --pyc 0 --no-extra --steps 2 --warmup 3 \
      2>&1 | tail -1 > gpurun_out/big_c5_$sc.json
    python -c "import json; d=json.load(open('gpurun_out/big_c5_$sc.json')); print('c5 $sc', d['config']['schedule'], d['config']['slots'], round(d['value']), d['kernel_ms'], d['parity']['mismatches'], d['gpu_launches'])" \
      | tee -a gpurun_out/split_big.txt
  done
  timeout 1200 python bench.py --workload c4 --schedule input+split --slots 45000 --arena-bytes 2621440 --no-cpu --pyc 0 --no-extra --steps 1 --warmup 1 \
    2>&1 | tail -1 > gpurun_out/big_c4_split.json
  python -c "import json; d=json.load(open('gpurun_out/big_c4_split.json')); print('c4 input+split', d['config']['slots'], round(d['value']), d['kernel_ms'], d['parity']['mismatches'], d['gpu_launches'])" \
    | tee -a gpurun_out/split_big.txt
}
split3() {  # schedule 4 (analyze | structure | emit kernels) vs 3 (tree | emit): parity + timing
  UPY_SCHEDULE=cost+split3 timeout 1500 python -m pytest -m gpu -x -q tests/test_golden_gpu.py tests/test_cli.py \
    2>&1 | tail -3 | tee gpurun_out/pytest_split3.txt
  for wl in c3 c3_311 c2x; do
    for sc in split split3 split split3; do
      o=cost; [ $wl = c2x ] && o=input
      timeout 900 python bench.py --workload $wl --schedule $o+$sc --no-cpu --pyc 0 --no-extra --steps 3 --warmup 2 \
        2>&1 | tail -1 > gpurun_out/s3_${wl}_$sc.json
      python -c "import json; d=json.load(open('gpurun_out/s3_${wl}_$sc.json')); print('$wl $sc', round(d['value']), d['kernel_ms'], d['parity']['mismatches'])" \
        | tee -a gpurun_out/split3.txt
    done
  done
}
c5() {  # one 16M-object corpus on this GPU (strong-scaling shape at N=1) + torchrun N=1 lines
  timeout 1800 python bench.py --workload c5 --no-cpu --pyc 0 --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_c5.json
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --gpus 1 --no-extra --no-cpu 2>&1 | tail -1 > gpurun_out/bench_torchrun1.json
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 \
    bench.py --impl reference --gpus 1 2>&1 | tail -1 > gpurun_out/bench_ref_torchrun1.json
}
for f in "$@"; do $f; done
