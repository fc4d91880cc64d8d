# column kernel: neighbour-column L1 prefetch variants
python tools/sweep.py 4x3_base 4x3_nbr 4x3_nbr1 4x3_nbr2 4x3_base 4x3_nbr 4x3_nbr1 4x3_nbr2 > gpurun_out/sweep_nbr.log 2>&1
cat gpurun_out/sweep_nbr.log
