python build_pb.py > gpurun_out/build.log 2>&1 || exit 1
PYTHONPATH=. PB_TC_DEBUG=10 timeout -s KILL 60 python scripts/timeline.py --calls 4 --out gpurun_out/tl10.npy > /dev/null 2>&1
python - <<'PY'
import numpy as np
rec=np.load('gpurun_out/tl10.npy')
k2=rec[rec[:,0]==2]; k5=rec[rec[:,0]==5]
d2={}; d5={}
for r in k2:
    if r[1] not in d2 or r[4]>d2[r[1]][4]: d2[r[1]]=r
for r in k5:
    if r[1] not in d5 or r[2]>d5[r[1]][2]: d5[r[1]]=r
first=[]; second=[]
for c in d2:
    r2=d2[c]; r5=d5[c]
    first.append((r5[3]-r2[5])/1e3)    # max done -> first chunk pass done (t_c0s[1])
    second.append((r2[6]-r5[2])/1e3)   # second pass start (t_c0s[0]) -> chunk0 done (tc0)
print("chunk0 build, first (cold) run: med %.2f us; second (warm) run: med %.2f us" % (np.median(first), np.median(second)))
PY
