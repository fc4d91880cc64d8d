timeout 900 python -m pytest tests/test_mover_gpu.py tests/test_field_gpu.py tests/test_moments_gpu.py -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do python bench.py --e2e-steps 0 --cpu-baseline 0 --strict-too 0 --strong 0 --general-3d 0 > gpurun_out/bench_q$i.log 2>/dev/null
python3 -c "
import json; d=json.loads(open('gpurun_out/bench_q$i.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['ms_per_step']-d['roofline']['kernel_ms'], d['gpu_launches'])"; done
