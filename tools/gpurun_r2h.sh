python tools/sweep.py 4x3_base 4x3_ur 4x3_base 4x3_ur > gpurun_out/sweep_ur.log 2>&1
cat gpurun_out/sweep_ur.log
