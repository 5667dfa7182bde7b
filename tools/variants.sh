#!/bin/bash
# Build alternative libedgebatch_b200.so variants of eb_dftsp.cu (extra nvcc
# defines) next to the in-tree objects, for A/B timing on the GPU box:
#   tools/variants.sh NAME "-DFOO=1 -DBAR=2" [NAME2 "DEFS2" ...]
# -> build/variants/NAME.so ; run with EB_LIB_PATH=build/variants/NAME.so
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2405_07140_b200._build import build_library; build_library()"
mkdir -p build/variants
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-ffp-contract=off -I include"
OTHERS=$(ls build/obj/*.o | grep -v eb_dftsp.o)
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  ( nvcc $F $defs -Xptxas -v -c -o build/variants/$name.o paper_2405_07140_b200/csrc/eb_dftsp.cu 2> build/variants/$name.ptxas \
    && nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/$name.so build/variants/$name.o $OTHERS \
    && echo "$name: $(grep -A2 'dftsp_lock_kernelILb1ELb0ELb0ELi1E' build/variants/$name.ptxas | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')" ) &
done
wait
