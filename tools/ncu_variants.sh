#!/bin/bash
# ncu --set full of the 3rd FAST mover launch, per lib variant (run on the GPU box).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  B2M_LIB=$PWD/paper_1904_03684_b200/libb2m_$v.so python tools/one_launch.py 3 || exit 1
  B2M_LIB=$PWD/paper_1904_03684_b200/libb2m_$v.so ncu --set full --import-source on --clock-control none \
    -k regex:warp_tile_kernel --launch-skip 2 --launch-count 1 -f -o gpurun_out/v_$v \
    python tools/one_launch.py 3 > gpurun_out/ncu_$v.log 2>&1 || { tail -5 gpurun_out/ncu_$v.log; exit 1; }
done
