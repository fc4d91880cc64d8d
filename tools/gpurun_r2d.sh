timeout 600 python -m pytest tests/test_moments_gpu.py -x -q 2>&1 | tail -2
PRESSURE=1 python tools/deposit_drift.py | cut -c1-40
python tools/cycle_c2.py --resort 4
