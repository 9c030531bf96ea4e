# interleaved comparison of prebuilt libraries scripts/libpb_<tag>.so for tags in $SO_TAGS (8-call graphs)
cp paper_2003_00822_b200/libpb.so /tmp/libpb_keep.so
for rep in 1 2; do
  for v in $SO_TAGS; do
    cp scripts/libpb_$v.so paper_2003_00822_b200/libpb.so; touch paper_2003_00822_b200/libpb.so
    echo "== [$rep] $v"
    for args in ${SO_AB_SHAPES:-"--L 2 8 16"}; do PYTHONPATH=. timeout -s KILL 300 python scripts/sweep_L.py ${args//,/ } 2>&1 | tail -1; done
  done
done
cp /tmp/libpb_keep.so paper_2003_00822_b200/libpb.so
