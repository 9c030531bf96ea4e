"""GPU layer helpers (FC / RNN / LSTM steps) against the oracle
composed with double-precision elementwise math (reading G15)."""
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


def _qw(pb, orc, W, L):
    w = pb.PackedWeights.quantize(W, L)
    codes, s, off, _ = orc.quantize_weights(W, L, "grid")
    assert w.scale == s
    return w, codes, s


@pytest.mark.parametrize("fn,name", [(1, "relu"), (2, "tanh"), (3, "sigmoid"), (0, "none")])
def test_linear(pb, torch, orc, fn, name):
    R, K, B, L, a = 1024, 784, 3, 4, 16
    W = synth.weights(R, K, 1)
    b = synth.bias(R, 2)
    x = synth.activations(B, K, 3, "mnist")
    w, codes, s = _qw(pb, orc, W, L)
    y = pb.linear(torch.from_numpy(x).cuda(), w, torch.from_numpy(b).cuda(), fn, L, a).cpu().numpy()
    _, yo, _ = orc.pbatch(codes, L, 0, s, L, x, a)
    z = yo.astype(np.float64) + b.astype(np.float64)
    ref = {"relu": np.maximum(z, 0), "tanh": np.tanh(z), "sigmoid": 1 / (1 + np.exp(-z)), "none": z}[name]
    np.testing.assert_allclose(y, ref, rtol=1e-5, atol=1e-6)


def test_mlp_forward(pb, torch, orc):
    # MNIST 3-layer MLP 784->1024->1024->10 (BASELINE config 2), ReLU between
    dims = [(1024, 784), (1024, 1024), (10, 1024)]
    x = synth.activations(1, 784, 10, "mnist")
    h_gpu = torch.from_numpy(x).cuda()
    h_or = x
    for li, (R, K) in enumerate(dims):
        W = synth.weights(R, K, 20 + li)
        b = synth.bias(R, 30 + li)
        L = [4, 2, 2][li]
        w, codes, s = _qw(pb, orc, W, L)
        fn = 1 if li < 2 else 0
        h_gpu = pb.linear(h_gpu, w, torch.from_numpy(b).cuda(), fn, L, 8)
        _, yo, _ = orc.pbatch(codes, L, 0, s, L, h_or, 8)
        z = yo.astype(np.float32) + b
        h_or = np.maximum(z, 0) if fn else z
        # compare layer by layer on the SAME input so the next layer is exact
        np.testing.assert_allclose(h_gpu.cpu().numpy(), h_or, rtol=1e-5, atol=1e-6)
        h_gpu = torch.from_numpy(h_or.astype(np.float32)).cuda()


@pytest.mark.parametrize("B,H,E,L_ih,L_hh", [(1, 256, 256, 4, 2), (4, 512, 300, 8, 8), (16, 128, 128, 1, 1)])
def test_lstm_step(pb, torch, orc, B, H, E, L_ih, L_hh):
    s = synth.seed(3, H + B)
    Wih = synth.weights(4 * H, E, s)
    Whh = synth.weights(4 * H, H, s + 1)
    bih, bhh = synth.bias(4 * H, s + 2), synth.bias(4 * H, s + 3)
    x = synth.activations(B, E, s + 4, "gauss")
    h = synth.activations(B, H, s + 5, "tanh")
    c = synth.activations(B, H, s + 6, "gauss")
    mode = "binary" if L_ih == 1 else "grid"
    qm = pb.PB_Q_BINARY if L_ih == 1 else pb.PB_Q_GRID
    wih = pb.PackedWeights.quantize(Wih, L_ih, qm)
    whh = pb.PackedWeights.quantize(Whh, L_hh, qm)
    ci, si, oi, _ = orc.quantize_weights(Wih, L_ih, mode)
    ch, sh, oh, _ = orc.quantize_weights(Whh, L_hh, mode)
    T = lambda a: torch.from_numpy(a).cuda()
    hn, cn = pb.lstm_step(T(x), T(h), T(c), wih, whh, T(bih), T(bhh), act_bits=16)
    _, yi, _ = orc.pbatch(ci, L_ih, oi, si, L_ih, x, 16)
    _, yh, _ = orc.pbatch(ch, L_hh, oh, sh, L_hh, h, 16)
    gates = yi.astype(np.float64) + bih + yh.astype(np.float64) + bhh
    h_ref, c_ref = orc.lstm_cell(gates, c)
    np.testing.assert_allclose(cn.cpu().numpy(), c_ref, rtol=1e-5, atol=2e-6)
    np.testing.assert_allclose(hn.cpu().numpy(), h_ref, rtol=1e-5, atol=2e-6)


def test_rnn_step(pb, torch, orc):
    B, H, E, L = 2, 512, 784, 6
    Wih, Whh = synth.weights(H, E, 1), synth.weights(H, H, 2)
    bih, bhh = synth.bias(H, 3), synth.bias(H, 4)
    x, h = synth.activations(B, E, 5), synth.activations(B, H, 6, "tanh")
    wih, whh = pb.PackedWeights.quantize(Wih, L), pb.PackedWeights.quantize(Whh, L)
    ci, si, _, _ = orc.quantize_weights(Wih, L)
    ch, sh, _, _ = orc.quantize_weights(Whh, L)
    T = lambda a: torch.from_numpy(a).cuda()
    hn = pb.rnn_step(T(x), T(h), wih, whh, T(bih), T(bhh), k_used_ih=4, k_used_hh=5, act_bits=16)
    _, yi, _ = orc.pbatch(ci, L, 0, si, 4, x, 16)
    _, yh, _ = orc.pbatch(ch, L, 0, sh, 5, h, 16)
    ref = np.tanh(yi.astype(np.float64) + bih + yh.astype(np.float64) + bhh)
    np.testing.assert_allclose(hn.cpu().numpy(), ref, rtol=1e-5, atol=2e-6)


def test_cuda_graph_capture(pb, torch, orc):
    # the call is stream-ordered, allocation- and sync-free: graph-capturable
    R, K, L = 2048, 2048, 8
    m = synth.codes(R, K, L, 77)
    w = pb.PackedWeights.from_codes(m, L, 0, 0.5)
    x = torch.from_numpy(synth.activations(1, K, 78)).cuda()
    ws = pb.Workspace(pb.workspace_bytes(1, K, 16))
    y = torch.empty(1, R, device="cuda")
    acc = torch.empty(1, R, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pb.matmul(x, w, L, 16, y=y, acc=acc, ws=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        pb.matmul(x, w, L, 16, y=y, acc=acc, ws=ws, stream=s)
    y.zero_()
    acc.zero_()
    g.replay()
    torch.cuda.synchronize()
    acc_o, y_o, _ = orc.pbatch(m, L, 0, 0.5, L, x.cpu().numpy(), 16)
    assert np.array_equal(acc.cpu().numpy(), acc_o)
    assert np.array_equal(y.cpu().numpy(), y_o)
