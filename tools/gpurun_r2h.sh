python tools/sweep.py 4x3_base 4x3_defer 4x3_base:3d 4x3_defer:3d 4x3_base 4x3_defer > gpurun_out/sweep_defer.log 2>&1
for v in base defer; do echo "== $v"; B2M_LIB=$PWD/paper_1904_03684_b200/libb2m_4x3_$v.so python tools/fused_time.py 2; done >> gpurun_out/sweep_defer.log 2>&1
cat gpurun_out/sweep_defer.log
