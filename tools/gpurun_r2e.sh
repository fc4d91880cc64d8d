mkdir -p /tmp/w1; python tests/nccl_world_worker.py 0 1 29555 /tmp/w1 2 ok; ls /tmp/w1; cat /tmp/w1/*.err 2>/dev/null
python -m pytest tests/test_world_nccl_gpu.py tests/test_world_gpu.py -q 2>&1 | tail -3
python bench.py > gpurun_out/bench3.log 2>&1; tail -1 gpurun_out/bench3.log
