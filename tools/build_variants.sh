#!/bin/bash
# Build in-tree variants of libb2m.so for tuning sweeps (tools/sweep.py):
#   TAG=_x EXTRA="-DB2M_..." tools/build_variants.sh PPTxMINBLOCKS ...
set -e
cd "$(dirname "$0")/../paper_1904_03684_b200/csrc"
for v in "$@"; do
  ppt=${v%%x*}; mb=${v##*x}
  obj=../../build/variant_$v$TAG; mkdir -p $obj
  objs=""
  for src in *.cu; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
         -I../../include -I. --expt-relaxed-constexpr \
         -DB2M_FAST_MINBLOCKS=$mb -DB2M_FAST_PPT=$ppt $EXTRA -c -o $obj/${src%.cu}.o $src &
    objs="$objs $obj/${src%.cu}.o"
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libb2m_$v$TAG.so $objs \
       ../../build/b2m/b2m_gem.o -Xcompiler -pthread -ldl
done
