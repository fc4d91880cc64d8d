for lib in libb2m.so libb2m_4x3_xfast.so; do
  echo "== $lib"; B2M_LIB=paper_1904_03684_b200/$lib python tools/deposit_drift.py
done
