# device-driven loop variants (ab_libs/*) vs the in-tree build, C2, interleaved
LIB=paper_2402_09222_b200/libomcg.so
cp $LIB /tmp/libomcg_head.so
for r in 1 2; do
  cp /tmp/libomcg_head.so $LIB
  for ds in 0 1; do echo "== head ds=$ds"; timeout 300 python scripts/run_c2.py 7 2 device_schedule=$ds 2>&1 | grep prof=0; done
  for v in "$@"; do cp ab_libs/$v/libomcg.so $LIB; echo "== $v ds=1"; timeout 300 python scripts/run_c2.py 7 2 device_schedule=1 2>&1 | grep prof=0; done
done
cp /tmp/libomcg_head.so $LIB
