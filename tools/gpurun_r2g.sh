g++ -std=c++17 -O2 -fPIC -shared -o /tmp/libfakenccl.so tests/fake_nccl/fake_nccl.cpp -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart -lrt
export B2M_NCCL_LIB=/tmp/libfakenccl.so B2M_DIST_BACKEND=gloo B2M_NATIVE_WORLD=force
timeout 1500 python bench.py --gpus ${NR:-2} --steps 4 --warmup 3 --e2e-steps 1 --cpu-baseline 0 > gpurun_out/bench_fake2.log 2> gpurun_out/bench_fake2.err; echo rc=$?
python3 -c "
import json; d=json.loads(open('gpurun_out/bench_fake2.log').read().strip().splitlines()[-1])
print(d['n_gpus'], d['value'], d['config']['parallelism'], d['verify'], d['counts_conserved'])
print(json.dumps(d['ranks'])); print(json.dumps(d['strong_scaling'])[:400]); print(json.dumps(d['c3'])[:400])"
grep -v "NCCL INFO" gpurun_out/bench_fake2.err | tail -5
