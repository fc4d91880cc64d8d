timeout 1500 python -m pytest tests/test_world_gpu.py tests/test_world_nccl_gpu.py tests/test_partition_gpu.py tests/test_mover_gpu.py -m gpu -x -q > gpurun_out/pt_world.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_world.log
B2M_BENCH_WORLD=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --steps 20 --warmup 5 --e2e-steps 0 --cpu-baseline 0 > gpurun_out/w1_lm.log 2>gpurun_out/w1_lm.err
python3 -c "
import json; d=json.loads(open('gpurun_out/w1_lm.log').read().strip().splitlines()[-1])
r=d.get('ranks',[{}])[0]
print('world1', d['ms_per_step'], r.get('mover_ms'), r.get('exchange_ms'), d.get('verify',{}).get('ok'), d.get('counts_conserved'))"
