# interleaved comparison of prebuilt libraries scripts/libpb_<V>.so for V in $SO_VARIANTS (8-call graphs)
cp paper_2003_00822_b200/libpb.so /tmp/libpb_keep.so
for rep in 1 2; do
  for v in ${SO_VARIANTS:-A B}; do
    cp scripts/libpb_$v.so paper_2003_00822_b200/libpb.so; touch paper_2003_00822_b200/libpb.so
    echo "== [$rep] $v"
    PYTHONPATH=. timeout -s KILL 300 python scripts/sweep_L.py ${SO_AB_ARGS:---L 2 8} 2>&1 | tail -1
  done
done
cp /tmp/libpb_keep.so paper_2003_00822_b200/libpb.so
