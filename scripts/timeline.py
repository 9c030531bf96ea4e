"""Per-CTA timeline of the act + tensor-engine GEMM chain (PB_TC_DEBUG=6 must be
set in the environment): captures `calls` back-to-back pb_matmul calls in a CUDA
graph (as bench.py does), replays it, and saves pb_debug_timeline's records
(see include/pb.h) to --out (.npy)."""
import argparse
import numpy as np
import torch

import paper_2003_00822_b200 as pb

ap = argparse.ArgumentParser()
ap.add_argument("--R", type=int, default=16384)
ap.add_argument("--K", type=int, default=16384)
ap.add_argument("--L", type=int, default=8)
ap.add_argument("--k-used", type=int, default=0)
ap.add_argument("--B", type=int, default=1)
ap.add_argument("--calls", type=int, default=4)
ap.add_argument("--copies", type=int, default=2, help="weight copies rotated over (1: L2-hot when it fits)")
ap.add_argument("--out", default="gpurun_out/tl.npy")
ap.add_argument("--time", type=int, default=0, help="replay the graph this many times and print us per call")
args = ap.parse_args()
k_used = args.k_used or args.L
rng = np.random.default_rng(1)
codes = rng.integers(-(1 << (args.L - 1)), 1 << (args.L - 1), size=(args.R, args.K), dtype=np.int32)
w0 = pb.PackedWeights.from_codes(codes, args.L)
ws_ = [w0] + [w0.clone_to(torch.empty_like(w0.buf)) for _ in range(args.copies - 1)]
x = torch.randn(args.B, args.K, device="cuda")
ws = pb.Workspace(pb.workspace_bytes(args.B, args.K, 16))
y = torch.empty(args.B, args.R, device="cuda")
for w in ws_:
    pb.matmul(x, w, k_used, 16, y=y, ws=ws)
torch.cuda.synchronize()
pb.debug_timeline()
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for i in range(args.calls):
        pb.matmul(x, ws_[i % len(ws_)], k_used, 16, y=y, ws=ws)
torch.cuda.synchronize()
pb.debug_timeline()
g.replay()
torch.cuda.synchronize()
rec = pb.debug_timeline()
if rec is not None:
    np.save(args.out, rec)
    print("records", len(rec))
if args.time:
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(args.time):
        g.replay()
    ev1.record()
    torch.cuda.synchronize()
    print(f"us_per_call {ev0.elapsed_time(ev1) * 1e3 / (args.time * args.calls):.2f}")
