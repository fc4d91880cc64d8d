for lib in libb2m.so libb2m_4x3_nouvw.so libb2m.so libb2m_4x3_nouvw.so; do
  echo "== $lib"; B2M_LIB=paper_1904_03684_b200/$lib python tools/fused_time.py 4
done
timeout 600 python -m pytest tests/test_moments_gpu.py -x -q -k fused 2>&1 | tail -2
