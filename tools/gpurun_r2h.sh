python tools/sweep.py 4x3_base:3d 4x3_p3:3d 4x3_base:3d 4x3_p3:3d 4x3_base > gpurun_out/sweep_p3.log 2>&1
cat gpurun_out/sweep_p3.log
