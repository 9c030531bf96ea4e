"""Per-step timeline of the persistent LSTM kernel (PB_TC_DEBUG=6): medians over CTAs of
step start -> h_full -> B built -> MMAs done -> arrived (us, relative to each step's start)."""
import math, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2003_00822_b200 as pb
H, T, L, B = 2048, 8, int(os.environ.get("L", 4)), int(os.environ.get("B", 1))
rng = np.random.default_rng(1)
W = lambda: torch.from_numpy(pb.interleave_gates((rng.standard_normal((4 * H, H)) / math.sqrt(H)).astype(np.float32))).cuda()
wi, wh = pb.PackedWeights.quantize_device(W(), L), pb.PackedWeights.quantize_device(W(), L)
xs = torch.randn(T, B, H, device="cuda")
h0, c0 = torch.tanh(torch.randn(B, H, device="cuda")), torch.randn(B, H, device="cuda")
bi = torch.zeros(4 * H, device="cuda")
ws = pb.Workspace(pb.pb_lstm_seq_workspace_bytes(T, B, H, H, 16))
pb.lstm_seq(xs, h0, c0, wi, wh, bi, ws=ws)
torch.cuda.synchronize()
pb.debug_timeline()
pb.lstm_seq(xs, h0, c0, wi, wh, bi, ws=ws)
torch.cuda.synchronize()
rec = pb.debug_timeline()
r = rec[rec[:, 0] == 7]
print("records", len(r))
for t in range(T):
    s = r[r[:, 2] == t]
    t0 = s[:, 3].min()
    f = lambda c: np.median((s[:, c] - t0) / 1e3)
    mx = lambda c: ((s[:, c] - t0) / 1e3).max()
    print(f"step {t}: start->h_full {f(4):6.2f} (max {mx(4):6.2f})  B built {f(5):6.2f}  MMAs done {f(6):6.2f} (max {mx(6):6.2f})  arrived {f(8):6.2f} (max {mx(8):6.2f})  finishers {int(s[:,7].sum())}")
print("cycles (median over CTAs, steps >= 1): h_full->casts done", np.median(r[r[:,2]>0][:,7]),
      " ballots", np.median(r[r[:,2]>0][:,9] // 1000000), " digit writes", np.median(r[r[:,2]>0][:,9] % 1000000))
c = rec[rec[:, 0] == 8]
c = c[c[:, 2] > 0]
if len(c):
    names = ["digits", "B built", "d_full", "drained", "reduced", "casts", "pre-arrive"]
    for fin in (0, 1):
        s = c[np.isin(c[:, 1], r[(r[:, 7] == fin)][:, 1])]
        print(("leader " if fin else "other  ") + "  ".join(f"{n} {np.median(s[:, 3 + i]) / 1.965e3:5.2f}" for i, n in enumerate(names)) + " us after h_full (clock64)")
x = rec[rec[:, 0] == 9]
if len(x):
    for t in range(1, T):
        pub = x[(x[:, 2] == t - 1) & (x[:, 5] > 0)][:, 5]
        det = x[x[:, 2] == t]
        if len(pub) and len(det):
            p1 = pub.max()
            print(f"step {t}: publish spread {(pub.max()-pub.min())/1e3:5.2f} us; detect after last publish: "
                  f"min {(det[:,3].min()-p1)/1e3:5.2f} med {(np.median(det[:,3])-p1)/1e3:5.2f} max {(det[:,3].max()-p1)/1e3:5.2f} us; "
                  f"poll rounds med {np.median(det[:,4]):.0f} max {det[:,4].max()}")
z = rec[(rec[:, 0] == 10) & (rec[:, 2] > 0)]
z = z[z[:, 3] > 0]
if len(z):
    print("leader finalisation (us after h_full, clock64): gx " + "  ".join(
        f"{n} {np.median(z[:, 3 + i]) / 1.965e3:5.2f}" for i, n in enumerate(["gx", "dequant", "cell", "max"])))
