"""Time the LSTM-LM input projection alone (W_ih x for T steps, one batched call) vs the
whole pb_lstm_seq call (scratch helper)."""
import math, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2003_00822_b200 as pb
H, T = 2048, 32
rng = np.random.default_rng(1)
W = (rng.standard_normal((4 * H, H)) / math.sqrt(H)).astype(np.float32)
for L in (2, 4, 8):
    w = pb.PackedWeights.quantize_device(torch.from_numpy(pb.interleave_gates(W)).cuda(), L)
    x = torch.randn(T, H, device="cuda")
    y = torch.empty(T, 4 * H, device="cuda")
    ws = pb.Workspace(pb.workspace_bytes(T, H, 16))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pb.matmul(x, w, L, 16, y=y, ws=ws, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(8):
            pb.matmul(x, w, L, 16, y=y, ws=ws, stream=s)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); [g.replay() for _ in range(10)]; e1.record(); torch.cuda.synchronize()
    print(f"L={L}: projection 8192x2048 x {T} columns: {e0.elapsed_time(e1) * 1e3 / 80:.2f} us/call", flush=True)
