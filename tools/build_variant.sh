#!/bin/bash
# Build an A/B variant of libsmpm.so: tools/build_variant.sh NAME "-DFLAG=..."
# -> paper_2605_28525_b200/libsmpm_NAME.so (select with SMPM_LIB=libsmpm_NAME.so)
set -e
cd "$(dirname "$0")/../paper_2605_28525_b200/csrc"
out=build/v_$1; mkdir -p $out
for f in smpm_sim smpm_module; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $2 -c $f.cu -o $out/$f.o
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libsmpm_$1.so $out/smpm_sim.o $out/smpm_module.o -lcudart
