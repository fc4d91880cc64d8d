timeout 600 python -m pytest tests/test_moments_gpu.py -x -q 2>&1 | tail -2
for lib in libb2m.so libb2m_4x3_reg.so; do
  echo "== $lib"; PRESSURE=1 B2M_LIB=paper_1904_03684_b200/$lib python tools/deposit_drift.py | cut -c1-40
done
