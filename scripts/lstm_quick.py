"""LSTM-LM (H = E = 2048, T timesteps) us per timestep: persistent kernel vs per-step launches
(scratch helper; bench.py reports the same in lstm_lm)."""
import math, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2003_00822_b200 as pb
H, T = int(os.environ.get("H", 2048)), int(os.environ.get("T", 32))
rng = np.random.default_rng(1)
Wih = (rng.standard_normal((4 * H, H)) / math.sqrt(H)).astype(np.float32)
Whh = (rng.standard_normal((4 * H, H)) / math.sqrt(H)).astype(np.float32)
bb = (0.1 * rng.standard_normal(4 * H)).astype(np.float32)
for L, B in [tuple(map(int, c.split(','))) for c in os.environ.get("CFGS", "2,1 4,1 6,1 8,1 10,1 16,1 4,4 8,4 4,16").split()]:
    wi = pb.PackedWeights.quantize_device(torch.from_numpy(pb.interleave_gates(Wih)).cuda(), L)
    wh = pb.PackedWeights.quantize_device(torch.from_numpy(pb.interleave_gates(Whh)).cuda(), L)
    xs = torch.randn(T, B, H, device="cuda")
    h0, c0 = torch.tanh(torch.randn(B, H, device="cuda")), torch.randn(B, H, device="cuda")
    bi = torch.from_numpy(pb.interleave_gates(bb)).cuda()
    ws = pb.Workspace(pb.pb_lstm_seq_workspace_bytes(T, B, H, H, 16))
    hs, cl = torch.empty(T, B, H, device="cuda"), torch.empty(B, H, device="cuda")
    out = []
    for mode in ("1", "0"):
        os.environ["PB_LSTM_PERSIST"] = mode
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            pb.lstm_seq(xs, h0, c0, wi, wh, bi, h_seq=hs, c_last=cl, ws=ws, stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            pb.lstm_seq(xs, h0, c0, wi, wh, bi, h_seq=hs, c_last=cl, ws=ws, stream=s)
        for _ in range(3): g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); [g.replay() for _ in range(10)]; e1.record(); torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3 / 10 / T)
    print(f"H={H} L={L} B={B}: persistent {out[0]:.2f} us/step, per-step launches {out[1]:.2f} us/step", flush=True)
