"""Repeat the C4 (16384x4096, L=8, B=128) parity check N times; print mismatching (b, row)
positions and their differences (scratch helper for an intermittent mismatch)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2003_00822_b200 as pb, oracle as orc, synth
R, K, L, a, B = 16384, 4096, 8, 16, int(os.environ.get("B", 128))
W = synth.weights_rows(R, K, synth.seed(4, 0))
x = synth.activations(B, K, synth.seed(4, 1), "gauss")
w = pb.PackedWeights.quantize(W, L, pb.PB_Q_GRID)
codes, s, off, _ = orc.quantize_weights(W, L, "grid")
rows = np.arange(0, R, 97)
acc_o, _, _ = orc.pbatch(codes[rows], L, off, s, L, x, a, nthreads=16)
xd = torch.from_numpy(x).cuda()
ws = pb.Workspace(pb.workspace_bytes(B, K, a))
acc = torch.zeros((B, R), dtype=torch.int64, device="cuda")
y = torch.empty((B, R), device="cuda")
bad = 0
for it in range(int(os.environ.get("N", 20))):
    pb.matmul(xd, w, L, a, y=y, acc=acc, ws=ws)
    torch.cuda.synchronize()
    g = acc.cpu().numpy()[:, rows]
    d = np.argwhere(g != acc_o)
    if len(d):
        bad += 1
        rr = rows[d[:, 1]]
        print(f"iter {it}: {len(d)} mismatches; rows {sorted(set(rr.tolist()))[:12]} tiles {sorted(set((rr // 128).tolist()))[:12]} "
              f"cols {sorted(set(d[:, 0].tolist()))[:20]} diff {[(int(g[i, j]) - int(acc_o[i, j])) for i, j in d[:6]]}", flush=True)
print("bad iterations", bad)
