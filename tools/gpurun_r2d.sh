for lib in libb2m.so libb2m_4x3_u3d2.so libb2m.so libb2m_4x3_u3d2.so; do
  echo "== $lib"; SW_3D=1 B2M_LIB=paper_1904_03684_b200/$lib python tools/one_launch.py 8 | tail -3
done
