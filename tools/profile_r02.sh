#!/bin/bash
# Round-2 evidence for profiles/ (run on the GPU box after the same commands ran clean):
#   launch list of a short bench run; ncu --set full of the FAST column mover
#   (DIM 2, the headline), the general FAST mover (DIM 3, z-varying field),
#   the STRICT column mover, the fused mover+deposit, and the deposit.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 0 \
    --strict-too 0 --cpu-baseline 0 --strong 0 --general-3d 0 > gpurun_out/ncu_bench.log 2>&1
echo "launches rc=$?"
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
$NCU -k "regex:warp_tile_kernel<(.int.)?4, (.bool.)?(0|false), (.int.)?2, (.bool.)?(0|false)>" \
    --launch-skip 2 --launch-count 1 -f -o gpurun_out/prof_col python tools/one_launch.py 3 \
    > gpurun_out/ncu_col.log 2>&1
echo "col rc=$?"
SW_3D=1 $NCU -k "regex:warp_tile_kernel<(.int.)?4, (.bool.)?(0|false), (.int.)?3, (.bool.)?(0|false)>" \
    --launch-skip 2 --launch-count 1 -f -o gpurun_out/prof_3d python tools/one_launch.py 3 \
    > gpurun_out/ncu_3d.log 2>&1
echo "3d rc=$?"
B2M_MODE=strict $NCU -k "regex:warp_tile_kernel<(.int.)?4, (.bool.)?(1|true), (.int.)?2" \
    --launch-skip 2 --launch-count 1 -f -o gpurun_out/prof_strict python tools/one_launch.py 3 \
    > gpurun_out/ncu_strict.log 2>&1
echo "strict rc=$?"
$NCU -k "regex:warp_tile_kernel<(.int.)?[0-9], (.bool.)?(0|false), (.int.)?2, (.bool.)?(1|true)>" \
    --launch-skip 1 --launch-count 1 -f -o gpurun_out/prof_fused python tools/fused_time.py 2 \
    > gpurun_out/ncu_fused.log 2>&1
echo "fused rc=$?"
ncu --set full --import-source on --clock-control none -k regex:deposit_ \
    --launch-skip 4 --launch-count 1 -f -o gpurun_out/prof_deposit python tools/deposit_drift.py \
    > gpurun_out/ncu_deposit.log 2>&1
echo "deposit rc=$?"
