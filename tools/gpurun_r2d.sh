for lib in libb2m.so libb2m_4x3_tp.so libb2m.so libb2m_4x3_tp.so; do
  echo "== $lib"; B2M_LIB=paper_1904_03684_b200/$lib python tools/one_launch.py 8 | tail -3
done
