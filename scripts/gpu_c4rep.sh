# intermittent-mismatch hunt: c4_repeat.py against several prebuilt libraries
python build_pb.py > /dev/null 2>&1
cp paper_2003_00822_b200/libpb.so /tmp/keep.so
for v in ${SO_VARIANTS}; do
  cp scripts/libpb_$v.so paper_2003_00822_b200/libpb.so; touch paper_2003_00822_b200/libpb.so
  echo "== $v: $(PYTHONPATH=. N=${N:-200} B=${B:-128} timeout -s KILL 600 python scripts/c4_repeat.py 2>&1 | tail -${TAILN:-3} | tr '\n' ' ')"
done
cp /tmp/keep.so paper_2003_00822_b200/libpb.so
