timeout 1500 python -m pytest tests/test_world_gpu.py tests/test_world_nccl_gpu.py tests/test_partition_gpu.py -m gpu -x -q 2>&1 | tail -1
B2M_BENCH_WORLD=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --steps 20 --warmup 5 --e2e-steps 0 --cpu-baseline 0 > gpurun_out/w1_p.log 2>gpurun_out/w1_p.err
python3 -c "
import json; d=json.loads(open('gpurun_out/w1_p.log').read().strip().splitlines()[-1])
print('world1', d['ms_per_step'], d['config']['parallelism'], d.get('verify',{}).get('ok'))"
