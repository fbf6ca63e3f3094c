# On the GPU box: C2 FoM of each ab_libs/<variant> (and the in-tree build as
# "head"), interleaved over R rounds: bash scripts/ab_run.sh R variant...
R=$1; shift
LIB=paper_2402_09222_b200/libomcg.so
cp $LIB /tmp/libomcg_head.so
for r in $(seq $R); do
  for v in head "$@"; do
    if [ $v = head ]; then cp /tmp/libomcg_head.so $LIB; else cp ab_libs/$v/libomcg.so $LIB; fi
    echo "== $v round $r"; timeout 300 python scripts/run_c2.py 7 2 2>&1 | grep -v "^$" | head -2
  done
done
cp /tmp/libomcg_head.so $LIB
