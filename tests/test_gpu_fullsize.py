"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (pb_matmul, engine AUTO, zero-filled workspace reused across calls):
sampled output rows are recomputed one by one by the oracle (its Alg. 2 on
exactly those rows of the same quantised layer) and compared bit-exactly
(acc) / to 1e-5 relative (y, also bit-identical per G13)."""
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
    return torch


_W_CACHE = {}


def _weights(R, K, cfg):
    key = (R, K, cfg)
    if key not in _W_CACHE:
        _W_CACHE.clear()
        _W_CACHE[key] = synth.weights_rows(R, K, synth.seed(cfg, 0))
    return _W_CACHE[key]


def _check(pb, torch, orc, R, K, L, a, B, k_used, kind, cfg, rows_sample=48, mode="grid"):
    W = _weights(R, K, cfg)
    x = synth.activations(B, K, synth.seed(cfg, 1), kind)
    qm = {"grid": pb.PB_Q_GRID, "binary": pb.PB_Q_BINARY}[mode]
    w = pb.PackedWeights.quantize(W, L, qm)
    codes, s, off, _ = orc.quantize_weights(W, L, mode)
    assert w.scale == s and w.offset == off
    xd = torch.from_numpy(x).cuda()
    ws = pb.Workspace(pb.workspace_bytes(B, K, a))
    acc = torch.zeros((B, R), dtype=torch.int64, device="cuda")
    y = torch.empty((B, R), device="cuda")
    for _ in range(2):   # second call reuses the workspace (stream-K counters must be back at 0)
        pb.matmul(xd, w, k_used, a, y=y, acc=acc, ws=ws)
    torch.cuda.synchronize()
    rng = np.random.default_rng(cfg)
    rows = np.unique(np.concatenate([[0, R - 1, R // 2, 127, 128], rng.integers(0, R, rows_sample)]))
    acc_o, y_o, _ = orc.pbatch(codes[rows], L, off, s, k_used, x, a, nthreads=8)
    acc_g = acc.cpu().numpy()[:, rows]
    y_g = y.cpu().numpy()[:, rows]
    assert np.array_equal(acc_g, acc_o)
    np.testing.assert_allclose(y_g, y_o, rtol=1e-5, atol=0)
    assert np.array_equal(y_g.view(np.uint32), y_o.view(np.uint32))


def test_c5_fc_16384_L8(pb, torch, orc):
    # BASELINE configs[4] at the bench configuration (L = 8, a = 16, batch 1)
    _check(pb, torch, orc, 16384, 16384, 8, 16, 1, 8, "gauss", 5)


@pytest.mark.parametrize("L,k_used", [(2, 2), (4, 3), (16, 16)])
def test_c5_fc_16384_other_L(pb, torch, orc, L, k_used):
    _check(pb, torch, orc, 16384, 16384, L, 16, 1, k_used, "gauss", 5, rows_sample=16)


def test_c5_binary(pb, torch, orc):
    _check(pb, torch, orc, 16384, 16384, 1, 16, 1, 1, "gauss", 5, rows_sample=24, mode="binary")


def test_c1_mnist_fc(pb, torch, orc):
    _check(pb, torch, orc, 1024, 784, 4, 16, 1, 4, "mnist", 1, rows_sample=1024)


def test_c3_lstm_gate_matvec(pb, torch, orc):
    # 4H x H gate matvec, H = 2048, 16 bitlayers, batch 1 and 16 (configs[2])
    _check(pb, torch, orc, 8192, 2048, 16, 16, 1, 16, "tanh", 3, rows_sample=64)
    _check(pb, torch, orc, 8192, 2048, 16, 16, 16, 12, "tanh", 3, rows_sample=16)


def test_c4_nli_batch128(pb, torch, orc):
    # configs[3]: 16384 x 4096, batch 128 (batched bitlayer GEMM regime)
    _check(pb, torch, orc, 16384, 4096, 8, 16, 128, 8, "gauss", 4, rows_sample=64)
