# What the driver runs at round end, on the committed tree (outputs in gpurun_out/).
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final_build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee gpurun_out/final_smoke.txt
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 | tee gpurun_out/final_pytest.txt
timeout 1200 python bench.py 2>&1 | tail -1 > gpurun_out/final_bench.json
timeout 900 python bench.py --impl reference 2>&1 | tail -1 > gpurun_out/final_bench_ref.json
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 \
  bench.py --gpus 1 --no-extra 2>&1 | tail -1 > gpurun_out/final_bench_torchrun1.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 \
  bench.py --impl reference --gpus 1 2>&1 | tail -1 > gpurun_out/final_bench_ref_torchrun.json
ls -la gpurun_out
