python tools/sweep.py 4x3_base 4x3_tail 4x3_base 4x3_tail 4x3_base 4x3_tail > gpurun_out/sweep_tail.log 2>&1
cat gpurun_out/sweep_tail.log
