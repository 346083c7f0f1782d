# f4 GPU parity + per-stage profile of the decompile kernel.  Outputs in gpurun_out/.
mkdir -p gpurun_out
python -m paper_2403_13839_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -m gpu -x -q tests/test_disasm.py tests/test_cli.py 2>&1 | tail -8 | tee gpurun_out/pytest_disasm.txt
UPY_LIB=paper_2403_13839_b200/_variants/prof.so timeout 600 python tools/stage_prof.py c3_310 c3_311 2>&1 | tee gpurun_out/stage_prof_c3.txt
UPY_LIB=paper_2403_13839_b200/_variants/prof.so timeout 900 python tools/stage_prof.py c4_310 c4_311 --objects 16384 2>&1 | tee gpurun_out/stage_prof_c4.txt
