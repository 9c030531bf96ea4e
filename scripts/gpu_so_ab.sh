# interleaved A/B of two prebuilt libraries scripts/libpb_A.so, scripts/libpb_B.so (8-call graphs)
for rep in 1 2; do
  for v in A B; do
    cp scripts/libpb_$v.so paper_2003_00822_b200/libpb.so; touch paper_2003_00822_b200/libpb.so
    echo "== [$rep] $v"
    for args in ${SO_AB_SHAPES:-"--L 2 8 16"}; do PYTHONPATH=. timeout -s KILL 300 python scripts/sweep_L.py ${args//,/ } 2>&1 | tail -1; done
  done
done
cp scripts/libpb_B.so paper_2003_00822_b200/libpb.so
