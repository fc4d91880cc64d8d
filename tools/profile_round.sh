#!/bin/bash
# Evidence for profiles/ (run on the GPU box after the same commands ran clean):
#   launch list of a short bench run, and one `ncu --set full` capture each of
#   the FAST mover, the STRICT mover and the moment deposition at C2.
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 \
    --strict-too 0 > gpurun_out/ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:warp_tile_kernel \
    --launch-skip 2 --launch-count 1 -f -o gpurun_out/prof_fast python tools/one_launch.py 3 \
    > gpurun_out/ncu_fast.log 2>&1
B2M_MODE=strict ncu --set full --import-source on --clock-control none -k regex:warp_tile_kernel \
    --launch-skip 2 --launch-count 1 -f -o gpurun_out/prof_strict python tools/one_launch.py 3 \
    > gpurun_out/ncu_strict.log 2>&1
# species 0 right after a cell sort (FAST context)
ncu --set full --import-source on --clock-control none -k regex:deposit_ \
    --launch-skip 0 --launch-count 1 -f -o gpurun_out/prof_deposit python tools/deposit_drift.py \
    > gpurun_out/ncu_deposit.log 2>&1
echo profiles captured
