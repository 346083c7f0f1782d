#!/bin/bash
# Build a variant of the decompile kernel object into paper_2403_13839_b200/_variants/<name>.so
# (linked with the current decode/loader objects).  Select it at run time with UPY_LIB=<path>.
#   tools/build_variant.sh minb6 -DUPY_MINB=6
#   CICC_OPT=-O2 PTXAS_OPT=-O3 tools/build_variant.sh opt23     (optimisation levels)
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
P=$R/paper_2403_13839_b200
mkdir -p $P/_variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -diag-suppress 550 \
  -Xcicc ${CICC_OPT:--O3} -Xptxas ${PTXAS_OPT:--O1} "$@" -c -o $P/_variants/$name.o $P/csrc/upy.cu
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $P/_variants/$name.so \
  $(ls $P/_build/*.o | grep -v '/upy.o$') $P/_variants/$name.o
rm -f $P/_variants/$name.o
echo built $P/_variants/$name.so
