for lib in libb2m.so libb2m_4x3_dp1.so libb2m_4x3_dp3.so; do
  echo "== $lib"; B2M_LIB=paper_1904_03684_b200/$lib python tools/fused_time.py 4
done
