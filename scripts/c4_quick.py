import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_2003_00822_b200 as pb, synth
R, K = 16384, 4096
W = synth.weights_rows(R, K, 1)
for L in (8, 4):
    w = pb.PackedWeights.quantize(W, L)
    for B in (1, 8, 32, 128):
        x = torch.from_numpy(synth.activations(B, K, 2)).cuda()
        ws = pb.Workspace(pb.workspace_bytes(B, K, 16))
        y = torch.empty((B, R), device='cuda')
        for _ in range(3): pb.matmul(x, w, L, 16, y=y, ws=ws)
        torch.cuda.synchronize()
        n = 20
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(n): pb.matmul(x, w, L, 16, y=y, ws=ws)
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / n
        bitmacs = R * K * L * 16 * B
        print(f"C4 L={L} B={B}: {us:.1f} us  {bitmacs/us/1e6:.3e} bit-MAC/s")
