"""C4-shape timing breakdown (scratch): planes kernel alone, GEMM alone, whole matmul."""
import ctypes as C, os, sys, torch
sys.path.insert(0, '.')
import paper_2003_00822_b200 as pb, synth
R, K = int(os.environ.get("R", 16384)), int(os.environ.get("K", 4096))
W = synth.weights_rows(R, K, 1)
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n
for L in [int(v) for v in os.environ.get("LS", "8").split(",")]:
    w = pb.PackedWeights.quantize(W, L)
    for B in [int(v) for v in os.environ.get("BS", "8,128").split(",")]:
        x = torch.from_numpy(synth.activations(B, K, 2)).cuda()
        ws = pb.Workspace(pb.workspace_bytes(B, K, 16))
        y = torch.empty((B, R), device='cuda')
        s = torch.cuda.current_stream().cuda_stream
        act = lambda: pb.check(pb.pb_act_quantize(x.data_ptr(), B, K, 16, pb.PB_ACT_AUTO, ws.ptr, ws.nbytes, s))
        gem = lambda: pb.check(pb.pb_bitgemm(ws.ptr, ws.nbytes, B, C.byref(w.desc), L, 16, y.data_ptr(), None, None, 0, 0, s))
        mm = lambda: pb.matmul(x, w, L, 16, y=y, ws=ws)
        print(f"R={R} K={K} L={L} B={B}: act {t(act):.1f} us, gemm {t(gem):.1f} us, matmul {t(mm):.1f} us", flush=True)
