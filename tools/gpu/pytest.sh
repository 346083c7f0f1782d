# GPU tests (args: pytest selection, default the whole -m gpu tier).  Outputs in gpurun_out/.
mkdir -p gpurun_out
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest -m gpu -x -q "${@:-tests}" 2>&1 | tail -25 | tee gpurun_out/pytest_gpu.txt
