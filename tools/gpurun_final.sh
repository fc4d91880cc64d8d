# final round-2 evidence: bench line + reference arm on a fresh box first, then the GPU suite and smoke
python bench.py > gpurun_out/bench_final.log 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/ref_final.log 2> gpurun_out/ref_final.err; echo "ref rc=$?"
python3 -c "
import json; d=json.loads(open('gpurun_out/bench_final.log').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])
r=json.loads(open('gpurun_out/ref_final.log').read().strip().splitlines()[-1]); print('ref', r['value'], r['config']['same_config'], (r.get('reference_simulation') or {}).get('value'))"
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
