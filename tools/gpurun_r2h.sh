python tools/sweep.py 4x3_base:3d 4x3_pf3:3d 4x3_base:3d 4x3_pf3:3d > gpurun_out/sweep_pf3.log 2>&1
cat gpurun_out/sweep_pf3.log
