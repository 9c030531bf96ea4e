"""Local mode of the fused tensor-engine kernel (GPU parity against the oracle): layers of at
most one (128-row tile, 1024-column chunk) unit per SM, where every CTA builds its own chunk's
activation digits and applies the sign correction per chunk -- with 2-4 chunk
clusters, and with 8 chunks (no cluster) -- and, next to them, the shapes just past it (two
units per CTA, the grid-wide B path: a local build of the second chunk measured slower), with
ragged K, a row tail, batch 1 and 3, and repeated calls on one workspace."""
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


@pytest.mark.parametrize("R,K,L,B", [
    (8192, 2048, 8, 1),     # 128 units: one per CTA, 2-chunk clusters
    (4096, 4096, 4, 3),     # 128 units, 4-chunk clusters, batch 3
    (2048, 8192, 8, 1),     # 128 units, 8 chunks: global partial sums
    (2048, 16384, 8, 1),    # 256 units: two per CTA, grid-wide B (the N = 8 shard of C5)
    (2304, 16000, 6, 3),    # 288 units, ragged K (last chunk partial), batch 3
    (4000, 9000, 5, 1),     # 32 x 9 = 288 units, row tail, odd L
])
def test_local_mode_parity(pb, torch, orc, R, K, L, B):
    s = synth.seed(11, R + K + L + B)
    W = synth.weights_rows(R, K, s)
    x = synth.activations(B, K, s + 1, "gauss")
    w = pb.PackedWeights.quantize(W, L, pb.PB_Q_GRID)
    codes, sc, off, _ = orc.quantize_weights(W, L, "grid")
    xd = torch.from_numpy(x).cuda()
    ws = pb.Workspace(pb.workspace_bytes(B, K, 16))
    acc = torch.zeros((B, R), dtype=torch.int64, device="cuda")
    y = torch.empty((B, R), device="cuda")
    for _ in range(3):                       # the workspace must be left clean by every call
        pb.matmul(xd, w, L, 16, y=y, acc=acc, ws=ws)
    torch.cuda.synchronize()
    rng = np.random.default_rng(R + K)
    rows = np.unique(np.concatenate([[0, 127, 128, 1023, 1024, R // 2, R - 1], rng.integers(0, R, 40)]))
    acc_o, y_o, _ = orc.pbatch(codes[rows], L, off, sc, L, x, 16, nthreads=8)
    assert np.array_equal(acc.cpu().numpy()[:, rows], acc_o)
    assert np.array_equal(y.cpu().numpy()[:, rows].view(np.uint32), y_o.view(np.uint32))
