for lib in libb2m_4x3_dp3.so libb2m_4x3_dp6.so libb2m_4x3_dp16.so; do
  echo "== $lib"; B2M_LIB=paper_1904_03684_b200/$lib python tools/deposit_drift.py | cut -c1-40; B2M_LIB=paper_1904_03684_b200/$lib python tools/fused_time.py 3
done
