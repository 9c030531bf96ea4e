"""Back-to-back self-consistency of the tensor engine (GPU): many identical calls in a row, no
host sync between them, must give identical integer accumulators -- and the first must equal the
oracle on a row sample.  This is the check that exposed an intermittent A-operand corruption in the
wide batched path ("A TMEM-store hazard"): a few rows of one pass in 2-8% of C4
B = 128 calls.  Shapes: C4 (16384 x 4096, L = 8) at batch 128 (wide), 8 (narrow, split path) and 1
(fused path)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import build_pb
    build_pb.build()
    import paper_2003_00822_b200 as pb
    return pb


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def c4(pb):
    R, K, L = 16384, 4096, 8
    W = synth.weights_rows(R, K, synth.seed(4, 0))
    return W, pb.PackedWeights.quantize(W, L, pb.PB_Q_GRID), L


@pytest.mark.parametrize("B,calls", [(128, 48), (8, 64), (1, 64)])
def test_back_to_back_identical(pb, torch, orc, c4, B, calls):
    W, w, L = c4
    R, K = W.shape
    a = 16
    x = synth.activations(B, K, synth.seed(4, 1), "gauss")
    xd = torch.from_numpy(x).cuda()
    ws = pb.Workspace(pb.workspace_bytes(B, K, a))
    y = torch.empty((B, R), device="cuda")
    outs = []
    for _ in range(calls):
        acc = torch.empty((B, R), dtype=torch.int64, device="cuda")
        pb.matmul(xd, w, L, a, y=y, acc=acc, ws=ws)
        outs.append(acc)
    torch.cuda.synchronize()
    first = outs[0]
    bad = [i for i, o in enumerate(outs) if not torch.equal(o, first)]
    assert not bad, f"calls {bad[:8]} differ from call 0"
    codes, s, off, _ = orc.quantize_weights(W, L, "grid")
    rows = np.arange(0, R, 257)
    acc_o, _, _ = orc.pbatch(codes[rows], L, off, s, L, x, a, nthreads=8)
    assert np.array_equal(first.cpu().numpy()[:, rows], acc_o)
