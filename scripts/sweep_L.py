"""Quick us/call sweep over L (k_used = L) at one shape, weights rotating over
>= 2x L2 (as bench.py), one CUDA graph per copy.  Experiment helper only.
  python scripts/sweep_L.py --L 1 2 4 8 [--R 16384 --K 16384 --B 1 --a 16]"""
import argparse
import math

import numpy as np
import torch

import paper_2003_00822_b200 as pb

ap = argparse.ArgumentParser()
ap.add_argument("--R", type=int, default=16384)
ap.add_argument("--K", type=int, default=16384)
ap.add_argument("--B", type=int, default=1)
ap.add_argument("--a", type=int, default=16)
ap.add_argument("--L", type=int, nargs="+", default=[1, 2, 4, 8, 16])
ap.add_argument("--steps", type=int, default=64)
ap.add_argument("--act-frac", type=int, default=-1024, help="PB_ACT_AUTO (-1024) or a literal f")
ap.add_argument("--split", action="store_true", help="pb_act_quantize + pb_bitgemm instead of pb_matmul")
ap.add_argument("--per", type=int, default=8, help="calls per CUDA graph (back to back, PDL-chained)")
args = ap.parse_args()
l2 = torch.cuda.get_device_properties(0).L2_cache_size
x = torch.randn(args.B, args.K, device="cuda")
y = torch.empty(args.B, args.R, device="cuda")
ws = pb.Workspace(pb.workspace_bytes(args.B, args.K, args.a))
rng = np.random.default_rng(1)
s = torch.cuda.Stream()
out = []
for L in args.L:
    if L == 1:
        codes = (1 - 2 * rng.integers(0, 2, size=(args.R, args.K))).astype(np.int32)
    else:
        codes = rng.integers(-(1 << (L - 1)), 1 << (L - 1), size=(args.R, args.K), dtype=np.int32)
    w0 = pb.PackedWeights.from_codes(codes, L, offset=1 if L == 1 else 0)
    M = max(1, math.ceil(2 * l2 / w0.nbytes()))
    cp = [w0] + [w0.clone_to(torch.empty_like(w0.buf)) for _ in range(M - 1)]
    with torch.cuda.stream(s):
        for w in cp:
            pb.matmul(x, w, L, args.a, args.act_frac, y=y, ws=ws, stream=s)
    torch.cuda.synchronize()
    M = max(M, 2)
    while len(cp) < M:
        cp.append(w0.clone_to(torch.empty_like(w0.buf)))
    def call(w):
        if args.split:
            pb.check(pb.pb_act_quantize(x.data_ptr(), args.B, args.K, args.a, args.act_frac, ws.ptr, ws.nbytes,
                                        s.cuda_stream))
            pb.check(pb.pb_bitgemm(ws.ptr, ws.nbytes, args.B, pb.C.byref(w.desc), L, args.a, y.data_ptr(), None,
                                   None, 0, 0, s.cuda_stream))
        else:
            pb.matmul(x, w, L, args.a, args.act_frac, y=y, ws=ws, stream=s)
    with torch.cuda.stream(s):
        for w in cp:
            call(w)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for t in range(args.per):
            call(cp[t % M])
    reps = max(1, args.steps // args.per)
    for i in range(2):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for i in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * args.per)
    gs = [g]
    gbs = (L * args.R * args.K / 8 + 4 * args.B * (args.K + args.R)) / us / 1e3
    out.append(f"L={L}:{us:.1f}us/{gbs:.0f}GB/s")
    del gs, cp, w0
    torch.cuda.empty_cache()
print(f"R={args.R} K={args.K} B={args.B} a={args.a}  " + "  ".join(out), flush=True)
