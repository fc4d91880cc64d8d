export B2M_MODE=strict
python tools/sweep.py 4x3_base 4x3_sp 4x3_base:3d 4x3_sp:3d 4x3_base 4x3_sp > gpurun_out/sweep_sp.log 2>&1
cat gpurun_out/sweep_sp.log
