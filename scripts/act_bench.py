"""Time pb_act_quantize alone (steps a1+a2) for a few shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_00822_b200 as pb

for (B, K, a) in [(1, 16384, 16), (1, 784, 16), (1, 4096, 16), (16, 2048, 16), (128, 4096, 16), (1, 65536, 32)]:
    x = torch.randn(B, K, device="cuda")
    ws = pb.Workspace(pb.workspace_bytes(B, K, a))
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(10):
        pb.check(pb.pb_act_quantize(x.data_ptr(), B, K, a, pb.PB_ACT_AUTO, ws.ptr, ws.nbytes, s))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 200
    e0.record()
    for _ in range(n):
        pb.check(pb.pb_act_quantize(x.data_ptr(), B, K, a, pb.PB_ACT_AUTO, ws.ptr, ws.nbytes, s))
    e1.record()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            pb.check(pb.pb_act_quantize(x.data_ptr(), B, K, a, pb.PB_ACT_AUTO, ws.ptr, ws.nbytes,
                                        torch.cuda.current_stream().cuda_stream))
    g.replay(); torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(True), torch.cuda.Event(True)
    e2.record()
    for _ in range(10):
        g.replay()
    e3.record()
    torch.cuda.synchronize()
    print(f"B={B} K={K} a={a}: stream {e0.elapsed_time(e1) / n * 1e3:.2f} us/launch, graph {e2.elapsed_time(e3) / 200 * 1e3:.2f} us/launch")
