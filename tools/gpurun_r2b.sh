set -x
timeout 1200 python -m pytest tests/test_large_configs_gpu.py -x -q > gpurun_out/pytest_large.log 2>&1; echo "large rc=$?"
tail -5 gpurun_out/pytest_large.log
timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/bench_g2.log 2> gpurun_out/bench_g2.err; echo "g2 rc=$?"
tail -c 3000 gpurun_out/bench_g2.log
tail -20 gpurun_out/bench_g2.err
timeout 600 python tools/bench_c5.py --steps 5 > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"; tail -2 gpurun_out/c5.log
