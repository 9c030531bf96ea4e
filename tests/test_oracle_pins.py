"""Pins for the CPU oracle (oracle/pb_oracle.c) against what the paper and
mathematics fix -- never against the oracle itself.  CPU only.

Pins:
  P1  Supplement §1 worked example, tests/golden/.
  P2  two's-complement identity sum_i S_i W_i == m, exhaustive L<=8.
  P3  bit-serial sum == brute-force integer matmul of the quantised values.
  P4  k_used == floor-truncated code (reading G12).
  P5  L=1 binary == textbook sign(W) @ x_q; multi-layer k_used=1 == sign layer.
  P6  Q(W) closed forms and the |Q-W| <= d/2 bound;
      the Alg. 1 floor bound.
  P7  activation cast: 1.5*2^16 = 98304; exact rational check; AUTO
      never saturates.
  P8  convergence of y to float64 W@x as bitlayers are added (north star).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "supp1_worked_example.json")


@pytest.fixture(scope="module")
def gold():
    with open(GOLD) as fh:
        return json.load(fh)


# ----------------------------------------------------------------- P1
def test_supp1_weight_layers_and_scales(orc, gold):
    W = np.array(gold["W"], np.int32)
    L = gold["L"]
    layers = orc.decompose(W, L)
    assert layers.tolist() == gold["W_layers_P417"]
    assert [orc.weight_layer_scale(L, 0, i) for i in range(L)] == gold["S_P435"]
    # the printed two's-complement patterns
    for r in range(2):
        for c in range(2):
            pat = int(gold["W_twos_complement_P405"][r][c], 2)
            assert [(pat >> (L - 1 - i)) & 1 for i in range(L)] == [int(layers[i, r, c]) for i in range(L)]


def test_supp1_quantizers_reproduce_integer_W(orc, gold):
    # d = (4 - (-4)) / 2^3 = 1 -> Q(W) = W; Alg. 1: W_q = W*2^16, max_bit = 18, lo = 16.
    W = np.array(gold["W"], np.float32)
    for mode in ("grid", "alg1"):
        codes, s, off, st = orc.quantize_weights(W, gold["L"], mode)
        assert st == orc.OK and off == 0
        assert codes.tolist() == gold["W"]
        assert s == 1.0


def test_supp1_activation_planes(orc, gold):
    x = np.array([gold["x"]], np.float32)
    a = gold["a"]
    xq, f = orc.quantize_activation(x, a, act_frac=0)
    assert xq.tolist() == [gold["x"]] and f.tolist() == [0]
    planes = orc.transpose(xq, a)            # [B][a][K]
    assert planes[0].T.tolist() == gold["x_bitmatrix_P447"]
    assert [orc.plane_scale(a, j) for j in range(a)] == gold["S_x_P453"]
    for k, pat in enumerate(gold["x_twos_complement_P409"]):
        p = int(pat, 2)
        assert [(p >> (a - 1 - j)) & 1 for j in range(a)] == gold["x_bitmatrix_P447"][k]


def test_supp1_result(orc, gold):
    W = np.array(gold["W"], np.int32)
    x = np.array([gold["x"]], np.float32)
    acc, y, f = orc.pbatch(W, gold["L"], 0, 1.0, gold["L"], x, gold["a"], act_frac=0)
    assert acc.tolist() == [gold["Wx"]]
    assert y.tolist() == [[float(v) for v in gold["Wx"]]]
    acc1, _, _ = orc.pbatch(W, gold["L"], 0, 1.0, 1, x, gold["a"], act_frac=0)
    assert acc1.tolist() == [gold["derived_k_used_1"]["value"]]


# ----------------------------------------------------------------- P2
@pytest.mark.parametrize("L", list(range(1, 9)))
def test_twos_complement_exhaustive(orc, L):
    m = np.arange(-(1 << (L - 1)), 1 << (L - 1), dtype=np.int32)
    layers = orc.decompose(m, L).astype(np.int64)
    # independent: the paper's scales typed here, -2^(L-1), 2^(L-2), ..., 1
    S = np.array([-(1 << (L - 1))] + [1 << (L - 1 - i) for i in range(1, L)], np.int64)
    assert np.array_equal(S @ layers, m)


@pytest.mark.parametrize("L", [9, 12, 16])
def test_twos_complement_random(orc, L):
    m = synth.codes(1, 4096, L, synth.seed(0, L)).ravel()
    layers = orc.decompose(m, L).astype(np.int64)
    S = np.array([-(1 << (L - 1))] + [1 << (L - 1 - i) for i in range(1, L)], np.int64)
    assert np.array_equal(S @ layers, m)
    with pytest.raises(ValueError):
        orc.decompose(np.array([1 << (L - 1)], np.int32), L)      # out of range


@pytest.mark.parametrize("a", [1, 2, 3, 7, 8, 16, 31, 32])
def test_plane_identity(orc, a):
    rng = np.random.default_rng(a)
    xq = rng.integers(-(1 << (a - 1)), (1 << (a - 1)), size=(3, 77), dtype=np.int64)
    planes = orc.transpose(xq, a).astype(np.int64)
    T = np.array([-(1 << (a - 1))] + [1 << (a - 1 - j) for j in range(1, a)], np.int64)
    assert np.array_equal(np.einsum("j,bjk->bk", T, planes), xq)


# ----------------------------------------------------------------- P3/P4
def _brute(m, L, offset, k_used, xq):
    """Textbook integer matmul of the (floor-truncated) codes with x_q."""
    sh = L - k_used
    mt = (m.astype(np.int64) >> sh) << sh           # arithmetic shift = floor
    return xq.astype(np.int64) @ (mt + offset).T     # [B][R]


CASES = [  # (R, K, B, L, a)
    (5, 37, 3, 4, 16), (3, 1, 1, 2, 8), (7, 64, 2, 8, 8), (4, 130, 4, 16, 16),
    (6, 33, 1, 3, 32), (2, 200, 5, 12, 7), (9, 31, 2, 1, 16), (1, 96, 1, 16, 31),
    (3, 129, 3, 5, 3), (8, 17, 2, 6, 1),
]


@pytest.mark.parametrize("R,K,B,L,a", CASES)
def test_bitserial_equals_bruteforce(orc, R, K, B, L, a):
    s = synth.seed(0, R * 1000 + K)
    if L == 1:
        m, off = synth.binary_codes(R, K, s), 1
    else:
        m, off = synth.codes(R, K, L, s), 0
    x = synth.inject_edges(synth.activations(B, K, s + 1, "gauss"), s + 2)
    xq, f = orc.quantize_activation(x, a)
    for k_used in sorted({1, max(1, L // 2), L}):
        acc, y, f2 = orc.pbatch(m, L, off, 0.37, k_used, x, a)
        assert np.array_equal(f2, f)
        if L == 1:
            ref = xq @ m.astype(np.int64).T
        else:
            ref = _brute(m, L, 0, k_used, xq)
        assert np.array_equal(acc, ref), (k_used,)
        # dequant closed form: y = acc * s_w * 2^-f_b, one rounding to float32
        exact = np.array([[float(Fraction(int(acc[b, r])) * Fraction(0.37) / Fraction(2) ** int(f[b]))
                           for r in range(R)] for b in range(B)])
        assert np.allclose(y, exact, rtol=1e-7, atol=0)


def test_stepwise_equals_composed(orc):
    # decompose/quantize_activation/transpose/bitserial composed by hand == pbatch
    R, K, B, L, a = 6, 70, 3, 5, 12
    m = synth.codes(R, K, L, 11)
    x = synth.activations(B, K, 12, "tanh")
    layers = orc.decompose(m, L)
    xq, f = orc.quantize_activation(x, a)
    planes = orc.transpose(xq, a)
    acc1, y1 = orc.bitserial(layers, 0, 3, 0.5, planes, xq, f)
    acc2, y2, _ = orc.pbatch(m, L, 0, 0.5, 3, x, a)
    assert np.array_equal(acc1, acc2) and np.array_equal(y1, y2)


def test_batch_columns_independent(orc):
    # reading G14: a batched call equals B batch-1 calls bit-exactly
    R, K, B, L, a = 5, 90, 4, 6, 16
    m = synth.codes(R, K, L, 21)
    x = synth.activations(B, K, 22, "relu") * np.array([[1e-3], [1.0], [1e3], [7.0]], np.float32)
    acc, y, f = orc.pbatch(m, L, 0, 0.1, L, x, a)
    for b in range(B):
        acc_b, y_b, _ = orc.pbatch(m, L, 0, 0.1, L, x[b:b + 1], a)
        assert np.array_equal(acc_b[0], acc[b]) and np.array_equal(y_b[0], y[b])


# ----------------------------------------------------------------- P5
def test_binary_is_textbook_sign_matvec(orc):
    W = synth.weights(7, 100, 31)
    W[0, 0] = 0.0                                   # sign(0) = +1
    codes, v, off, st = orc.quantize_weights(W, 1, "binary")
    assert st == orc.OK and off == 1
    sgn = np.where(W < 0, -1, 1)
    assert np.array_equal(codes, sgn)
    assert v == pytest.approx(float(np.mean(np.abs(W.astype(np.float64)))), rel=1e-12)
    # v is the L2-optimal magnitude for W ~ u*sign(W): check against a sweep
    us = np.linspace(0.5 * v, 1.5 * v, 201)
    errs = [np.sum((W - u * sgn) ** 2) for u in us]
    assert abs(us[int(np.argmin(errs))] - v) <= (us[1] - us[0])
    x = synth.activations(2, 100, 32)
    xq, f = orc.quantize_activation(x, 16)
    acc, y, _ = orc.pbatch(codes, 1, 1, v, 1, x, 16)
    assert np.array_equal(acc, xq @ sgn.T.astype(np.int64))


@pytest.mark.parametrize("L", [2, 4, 8, 16])
def test_kused1_is_sign_layer(orc, L):
    m = synth.codes(6, 50, L, 40 + L)
    x = synth.activations(2, 50, 41)
    xq, _ = orc.quantize_activation(x, 16)
    acc, _, _ = orc.pbatch(m, L, 0, 1.0, 1, x, 16)
    assert np.array_equal(acc, -(1 << (L - 1)) * (xq @ (m < 0).T.astype(np.int64)))


# ----------------------------------------------------------------- P6
def test_quantize_round_closed_forms(orc):
    Q, d, st = orc.quantize_round(np.array([0.1, 0.4], np.float32), 2)
    assert d == pytest.approx(0.075, rel=1e-7)
    assert Q == pytest.approx([0.075, 0.375], rel=1e-6)
    # ties to even (reading G4): d = 1 -> 0.5 -> 0, 1.5 -> 2, 2.5 -> 2
    Q, d, _ = orc.quantize_round(np.array([0.0, 0.5, 1.5, 2.5, 4.0], np.float32), 2)
    assert d == 1.0 and Q.tolist() == [0.0, 0.0, 2.0, 2.0, 4.0]
    # a matrix already on the grid is a fixed point
    g = (np.arange(-8, 9, dtype=np.float32) * 0.125)   # span 2 = 2^4 * 0.125
    Q, d, _ = orc.quantize_round(g, 4)
    assert np.array_equal(Q, g.astype(np.float64))


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 15])
def test_quantize_round_error_bound(orc, n):
    W = synth.weights(16, 64, 50 + n)
    Q, d, _ = orc.quantize_round(W, n)
    assert d == pytest.approx((float(W.max()) - float(W.min())) / 2 ** n, rel=1e-12)
    assert np.max(np.abs(Q - W.astype(np.float64))) <= d / 2 * (1 + 1e-12)
    # grid codes reproduce Q where unclamped
    codes, s, _, _ = orc.quantize_weights(W, n + 1, "grid")
    lim = (1 << n) - 1
    inside = np.abs(codes) < lim
    assert np.array_equal(s * codes[inside], Q[inside])


def test_degenerate_weights(orc):
    z = np.zeros((3, 5), np.float32)
    codes, s, _, st = orc.quantize_weights(z, 4, "grid")
    assert st == orc.EDEGENERATE and not codes.any() and s == 1.0
    c = np.full((2, 3), -0.75, np.float32)
    codes, s, _, st = orc.quantize_weights(c, 4, "grid")
    assert st == orc.EDEGENERATE and s == 0.75 and (codes == -1).all()


@pytest.mark.parametrize("L", [2, 3, 4, 8])
def test_alg1_floor_bound(orc, L):
    W = synth.weights(8, 32, 60 + L)
    Q, d, _ = orc.quantize_round(W, L - 1)
    codes, s, _, st = orc.quantize_weights(W, L, "alg1")
    assert st == orc.OK
    assert codes.min() >= -(1 << (L - 1)) and codes.max() <= (1 << (L - 1)) - 1
    # floor(W_q / 2^lo) * 2^lo in (W_q - 2^lo, W_q], W_q = trunc(Q*2^16)
    err = s * codes - Q
    assert np.all(err <= 2.0 ** -16) and np.all(err > -(s + 2.0 ** -16))


# ----------------------------------------------------------------- P7
def test_activation_cast_closed_forms(orc):
    xq, f = orc.quantize_activation(np.array([[1.5]], np.float32), 32, act_frac=16)
    assert xq.tolist() == [[98304]] and f.tolist() == [16]
    xq, f = orc.quantize_activation(np.array([[1.0, -1.0]], np.float32), 8, act_frac=16)
    assert xq.tolist() == [[127, -128]]                                    # saturates
    xq, f = orc.quantize_activation(np.zeros((1, 4), np.float32), 16)
    assert f.tolist() == [0] and not xq.any()


@pytest.mark.parametrize("a", [1, 2, 8, 16, 31, 32])
def test_activation_auto_exact(orc, a):
    x = synth.inject_edges(synth.activations(3, 257, 70 + a), 71 + a)
    xq, f = orc.quantize_activation(x, a)
    for b in range(3):
        mx = max(abs(Fraction(float(v))) for v in x[b])
        if mx == 0:
            assert f[b] == 0 and not xq[b].any()
            continue
        # smallest e with max < 2^e, f = a-1-e  (reading G8)
        e = 0
        while not mx < Fraction(2) ** e:
            e += 1
        while mx < Fraction(2) ** (e - 1):
            e -= 1
        assert f[b] == a - 1 - e
        for c in range(0, 257, 7):
            v = Fraction(float(x[b, c])) * Fraction(2) ** int(f[b])
            assert xq[b, c] == int(v)                  # int() truncates toward zero
        assert np.abs(xq[b]).max() <= (1 << (a - 1)) - 1     # never saturates
        if a >= 2:
            assert np.abs(xq[b]).max() >= (1 << (a - 2))     # uses the top bit


# ----------------------------------------------------------------- P8
def test_convergence_to_float(orc):
    R, K = 64, 512
    W = synth.weights(R, K, 80)
    x = synth.activations(2, K, 81)
    ref = x.astype(np.float64) @ W.astype(np.float64).T
    errs = {}
    for L in (2, 4, 6, 8, 10, 12, 14, 16):
        codes, s, _, _ = orc.quantize_weights(W, L, "grid")
        _, y, _ = orc.pbatch(codes, L, 0, s, L, x, 32)
        errs[L] = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    Ls = sorted(errs)
    for l0, l1 in zip(Ls, Ls[1:]):
        assert errs[l1] < errs[l0]
        assert errs[l0] / errs[l1] > 2.5          # ~4x per 2 added layers
    assert errs[16] < 2e-4
    # activation floor: a=8 saturates the ladder
    codes, s, _, _ = orc.quantize_weights(W, 16, "grid")
    _, y8, _ = orc.pbatch(codes, 16, 0, s, 16, x, 8)
    e8 = np.linalg.norm(y8 - ref) / np.linalg.norm(ref)
    assert 1e-3 < e8 < 1e-1


def test_kused_ladder_monotone(orc):
    # truncating layers (floor) degrades monotonically on an ensemble
    R, K, L = 64, 256, 12
    W = synth.weights(R, K, 90)
    x = synth.activations(4, K, 91)
    ref = x.astype(np.float64) @ W.astype(np.float64).T
    codes, s, _, _ = orc.quantize_weights(W, L, "grid")
    prev = np.inf
    for k in range(2, L + 1):
        _, y, _ = orc.pbatch(codes, L, 0, s, k, x, 16)
        e = np.linalg.norm(y - ref)
        assert e < prev
        prev = e


def test_search_clip_property(orc):
    # parity unpinned (reading G6); property: never worse than no clipping
    W = np.concatenate([np.random.default_rng(5).uniform(-0.1, 0.1, 9999), [1.0]]).astype(np.float32)
    t, st = orc.search_clip(W, 5)
    assert st == orc.OK and t < 1.0

    def err(clip):
        codes, s, _, _ = orc.quantize_weights(W, 5, "grid", clip)
        return np.mean(np.abs(s * codes - W))
    assert err(t) <= err(1.0)


def test_midpoint_offset_identity_and_error(orc):
    """SURVEY §8(f) f4 midpoint option (not in the paper): with k_used < L the kept layers
    are the floor-truncated code (reading G12); the midpoint adds 2^(L-k_used-1) per code,
    i.e. acc gains exactly 2^(L-k_used-1) * sum_c x_q -- and, being the centre of the
    dropped range, lowers the error against the float product on Gaussian data."""
    import numpy as np
    import synth
    R, K, L = 64, 512, 8
    W = synth.weights(R, K, synth.seed(11, 0))
    x = synth.activations(3, K, synth.seed(11, 1), "gauss")
    codes, s, off, _ = orc.quantize_weights(W, L, "grid")
    for k in (1, 3, 5, 7):
        a0, y0, f = orc.pbatch(codes, L, off, s, k, x, 16)
        a1, y1, _ = orc.pbatch(codes, L, off, s, k, x, 16, midpoint=True)
        xq = np.trunc(np.ldexp(x.astype(np.float64), f[:, None])).astype(np.int64)   # exact cast (G8)
        np.testing.assert_array_equal(a1 - a0, np.broadcast_to((1 << (L - k - 1)) * xq.sum(axis=1)[:, None], a0.shape))
        ref = x.astype(np.float64) @ W.astype(np.float64).T
        e0 = np.abs(y0 - ref).mean()
        e1 = np.abs(y1 - ref).mean()
        assert e1 < e0, (k, e0, e1)
    a0, _, _ = orc.pbatch(codes, L, off, s, L, x, 16)
    a1, _, _ = orc.pbatch(codes, L, off, s, L, x, 16, midpoint=True)
    np.testing.assert_array_equal(a0, a1)          # k_used = L: nothing dropped, no offset


# ----------------------------------------------------------------- P9 (reading G15)
def test_lstm_cell_matches_torch_lstmcell(orc):
    # or_lstm_cell is pinned to PyTorch's nn.LSTMCell (reading G15: PyTorch nn.LSTM semantics,
    # gate order i, f, g, o; P:258 LSTM LM).  nn.LSTMCell computes its gates as
    # W_ih x + b_ih + W_hh h + b_hh; with W_ih = I (4H x 4H), W_hh = 0 and zero biases the gate
    # pre-activations are exactly x, so LSTMCell(x = gates, (h, c)) is the cell alone, in float64.
    # A swapped gate (e.g. i <-> f, or tanh on o) or a wrong update (c' = i c + f g) fails here.
    import torch
    B, H = 5, 37
    rng = np.random.default_rng(20200302)
    gates = rng.normal(0.0, 2.0, (B, 4 * H))
    gates[0, :] = 0.0                                     # sigmoid(0) = 1/2, tanh(0) = 0
    gates[1, :H] = 30.0                                   # saturated input gate
    c = rng.normal(0.0, 1.0, (B, H)).astype(np.float32)
    cell = torch.nn.LSTMCell(4 * H, H, bias=True, dtype=torch.float64)
    with torch.no_grad():
        cell.weight_ih.copy_(torch.eye(4 * H, dtype=torch.float64))
        cell.weight_hh.zero_()
        cell.bias_ih.zero_()
        cell.bias_hh.zero_()
        h_t, c_t = cell(torch.from_numpy(gates), (torch.zeros(B, H, dtype=torch.float64),
                                                   torch.from_numpy(c.astype(np.float64))))
    h_o, c_o = orc.lstm_cell(gates, c)
    np.testing.assert_allclose(c_o, c_t.numpy(), rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(h_o, h_t.numpy(), rtol=1e-13, atol=1e-15)
    # closed form at zero gates: c' = c / 2, h' = tanh(c / 2) / 2
    c0 = c[0].astype(np.float64)
    np.testing.assert_allclose(c_o[0], c0 / 2.0, rtol=1e-15)
    np.testing.assert_allclose(h_o[0], np.tanh(c0 / 2.0) / 2.0, rtol=1e-14)
