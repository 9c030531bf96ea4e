"""One pb_lstm_seq call (scratch, for compute-sanitizer): env H, T, L, B."""
import math, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2003_00822_b200 as pb
H, T, L, B = (int(os.environ.get(k, d)) for k, d in (("H", 2048), ("T", 3), ("L", 4), ("B", 16)))
rng = np.random.default_rng(1)
W = lambda: torch.from_numpy(pb.interleave_gates((rng.standard_normal((4 * H, H)) / math.sqrt(H)).astype(np.float32))).cuda()
wi, wh = pb.PackedWeights.quantize_device(W(), L), pb.PackedWeights.quantize_device(W(), L)
xs = torch.randn(T, B, H, device="cuda")
h0, c0 = torch.tanh(torch.randn(B, H, device="cuda")), torch.randn(B, H, device="cuda")
hs, cl = pb.lstm_seq(xs, h0, c0, wi, wh, torch.zeros(4 * H, device="cuda"))
torch.cuda.synchronize()
print("ok", float(hs.abs().max()))
