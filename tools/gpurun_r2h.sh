python tools/sweep.py 4x3_b:3d 4x4_b:3d 4x3_b:3d 4x4_b:3d > gpurun_out/sweep_mb.log 2>&1
cat gpurun_out/sweep_mb.log
