# world step at N=1: cost of the closing verdict all-reduce + host sync
for v in base nov base nov; do
  B2M_LIB=$PWD/paper_1904_03684_b200/libb2m_4x3_$v.so B2M_BENCH_WORLD=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --steps 20 --warmup 5 --e2e-steps 0 --cpu-baseline 0 > gpurun_out/w1_$v.log 2>gpurun_out/w1_$v.err
  python3 -c "
import json,sys; d=json.loads(open('gpurun_out/w1_$v.log').read().strip().splitlines()[-1])
r=d.get('ranks',[{}])[0]
print('$v', d['ms_per_step'], r.get('mover_ms'), r.get('exchange_ms'))"
done
