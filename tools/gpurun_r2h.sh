python tools/sweep.py 4x3_base:3d 4x3_3u2:3d 4x3_base:3d 4x3_3u2:3d > gpurun_out/sweep_3u.log 2>&1
cat gpurun_out/sweep_3u.log
