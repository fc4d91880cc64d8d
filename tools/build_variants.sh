#!/bin/bash
# Build in-tree variants of libb2m.so for tuning sweeps (tools/sweep.py).
set -e
cd "$(dirname "$0")/../paper_1904_03684_b200/csrc"
for v in "$@"; do
  ppt=${v%%x*}; mb=${v##*x}
  obj=../../build/variant_$v$TAG; mkdir -p $obj
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include -I. \
       -DB2M_FAST_PPT=$ppt -DB2M_FAST_MINBLOCKS=$mb $EXTRA -c -o $obj/k.o b2m_kernels.cu &
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include -I. \
       -DB2M_FAST_PPT=$ppt -DB2M_FAST_MINBLOCKS=$mb $EXTRA -c -o $obj/c.o b2m_capi.cu &
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libb2m_$v$TAG.so $obj/k.o $obj/c.o ../../build/b2m/b2m_gem.o -Xcompiler -pthread
done
