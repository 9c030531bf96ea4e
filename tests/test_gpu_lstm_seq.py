"""GPU parity of pb_lstm_seq (the input projection of all
timesteps hoisted into one batched call; the recurrence either as ONE persistent
tensor-engine kernel with a grid barrier per timestep (pb_lstm_tc.cu, default when
W_hh's units fit the SMs) or as one fused launch per timestep whose finalisation
applies the LSTM cell (PB_LSTM_PERSIST=0), reading G15) against
the CPU oracle, teacher-forced: step t is checked on the GPU's own h_t, c_t, so
every step is compared at the 1e-5 bar without drift.  A free-running run is
checked against the oracle's own 32-step recurrence with a drift bound."""
import os

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


@pytest.fixture(params=["persist", "per_step"])
def persist(request):
    old = os.environ.get("PB_LSTM_PERSIST")
    os.environ["PB_LSTM_PERSIST"] = "1" if request.param == "persist" else "0"
    yield request.param
    if old is None:
        del os.environ["PB_LSTM_PERSIST"]
    else:
        os.environ["PB_LSTM_PERSIST"] = old


@pytest.mark.parametrize("T,B,H,E,L_ih,L_hh,engine", [
    (5, 1, 256, 192, 3, 4, "auto"),      # fused cell, B = 1
    (4, 3, 128, 256, 8, 2, "auto"),      # batch 3 (N = 48 -> 64)
    (3, 8, 160, 128, 4, 4, "auto"),      # 2 batch slices per step, ragged H tile
    (2, 2, 64, 96, 1, 1, "auto"),        # binary weights (L = 1)
    (3, 2, 128, 96, 4, 4, "popc"),       # split path: planes + POPC GEMM + interleaved cell kernel
    (3, 2, 128, 2048, 16, 16, "auto"),   # hoisted W_ih with 2 accumulator groups (narrowed slices)
    (4, 1, 1100, 256, 4, 4, "auto"),     # W_hh K = 1100: 2 chunks, every tile split over 2 CTAs
    (3, 16, 512, 128, 4, 6, "auto"),     # batch 16: 128 digit columns (wide), 3 passes
    (3, 2, 2048, 256, 4, 4, "auto"),     # the LSTM-LM shape (H = 2048): 128 CTAs
    (3, 5, 300, 200, 5, 7, "auto"),      # odd L, ragged tiles, a 4-row tail tile; 4 passes: A of the
                                         # last in SMEM (persistent kernel)
    (4, 1, 2048, 256, 4, 8, "auto"),     # LSTM-LM shape, L = 8: 3 passes' A in TMEM + 1 in SMEM
    (3, 1, 512, 128, 4, 10, "auto"),     # L = 10: 2 passes' A in SMEM
    (3, 4, 256, 128, 4, 9, "auto"),      # odd L = 9, batch 4: the canonical last layer's A in SMEM
])
def test_lstm_seq(pb, torch, orc, persist, T, B, H, E, L_ih, L_hh, engine):
    s = synth.seed(7, T + 10 * B + H + E)
    Wih = synth.weights(4 * H, E, s)
    Whh = synth.weights(4 * H, H, s + 1)
    bias = (synth.bias(4 * H, s + 2) + synth.bias(4 * H, s + 3)).astype(np.float32)
    x = np.stack([synth.activations(B, E, s + 10 + t, "gauss") for t in range(T)])
    h0 = synth.activations(B, H, s + 4, "tanh")
    c0 = synth.activations(B, H, s + 5, "gauss")
    mode_i, mode_h = ("binary" if L_ih == 1 else "grid"), ("binary" if L_hh == 1 else "grid")
    qm = lambda m: pb.PB_Q_BINARY if m == "binary" else pb.PB_Q_GRID
    Wih_i, Whh_i, bias_i = pb.interleave_gates(Wih), pb.interleave_gates(Whh), pb.interleave_gates(bias)
    wih = pb.PackedWeights.quantize(Wih_i, L_ih, qm(mode_i))
    whh = pb.PackedWeights.quantize(Whh_i, L_hh, qm(mode_h))
    ci, si, oi, _ = orc.quantize_weights(Wih_i, L_ih, mode_i)
    ch, sh, oh, _ = orc.quantize_weights(Whh_i, L_hh, mode_h)
    D = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    c_seq = torch.empty((T, B, H), dtype=torch.float32, device="cuda")
    pb.set_engine({"auto": pb.PB_ENGINE_AUTO, "popc": pb.PB_ENGINE_POPC}[engine])
    try:
        ws = pb.Workspace(pb.pb_lstm_seq_workspace_bytes(T, B, E, H, 16))
        outs = []
        for rep in range(2):                    # the same workspace twice: self-cleaning scratch
            h_seq, c_last = pb.lstm_seq(D(x), D(h0), D(c0), wih, whh, D(bias_i), act_bits=16, c_seq=c_seq, ws=ws)
            torch.cuda.synchronize()
            outs.append((h_seq.cpu().numpy(), c_seq.cpu().numpy(), c_last.cpu().numpy()))
    finally:
        pb.set_engine(pb.PB_ENGINE_AUTO)
    hs, cs, cl = outs[0]
    assert np.array_equal(hs, outs[1][0]) and np.array_equal(cs, outs[1][1])
    assert np.array_equal(cl, cs[T - 1])
    for t in range(T):
        h_t = h0 if t == 0 else hs[t - 1]
        c_t = c0 if t == 0 else cs[t - 1]
        _, yi, _ = orc.pbatch(ci, L_ih, oi, si, L_ih, x[t], 16)
        _, yh, _ = orc.pbatch(ch, L_hh, oh, sh, L_hh, h_t, 16)
        g_ilv = yi.astype(np.float64) + bias_i + yh.astype(np.float64)        # [B][4H], interleaved rows
        g_gm = pb.deinterleave_gates(g_ilv.T).T                               # gate-major
        h_ref, c_ref = orc.lstm_cell(g_gm, c_t)
        np.testing.assert_allclose(cs[t], c_ref, rtol=1e-5, atol=2e-6, err_msg=f"c step {t}")
        np.testing.assert_allclose(hs[t], h_ref, rtol=1e-5, atol=2e-6, err_msg=f"h step {t}")


def test_lstm_seq_matches_lstm_step(pb, torch):
    """The fused sequence equals pb_lstm_step applied step by step (gate-major
    weights) up to fp32 rounding of the gate sums."""
    T, B, H, E, L = 3, 2, 128, 128, 4
    s = synth.seed(7, 999)
    Wih, Whh = synth.weights(4 * H, E, s), synth.weights(4 * H, H, s + 1)
    bih, bhh = synth.bias(4 * H, s + 2), synth.bias(4 * H, s + 3)
    x = np.stack([synth.activations(B, E, s + 10 + t, "gauss") for t in range(T)])
    h0, c0 = synth.activations(B, H, s + 4, "tanh"), synth.activations(B, H, s + 5, "gauss")
    D = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    wih_g, whh_g = pb.PackedWeights.quantize(Wih, L), pb.PackedWeights.quantize(Whh, L)
    wih_i = pb.PackedWeights.quantize(pb.interleave_gates(Wih), L)
    whh_i = pb.PackedWeights.quantize(pb.interleave_gates(Whh), L)
    h_seq, c_last = pb.lstm_seq(D(x), D(h0), D(c0), wih_i, whh_i,
                                D(pb.interleave_gates((bih + bhh).astype(np.float32))))
    h, c = D(h0), D(c0)
    for t in range(T):
        h, c = pb.lstm_step(D(x[t]), h, c, wih_g, whh_g, D(bih), D(bhh))
        np.testing.assert_allclose(h_seq[t].cpu().numpy(), h.cpu().numpy(), rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(c_last.cpu().numpy(), c.cpu().numpy(), rtol=1e-4, atol=1e-5)


def test_lstm_seq_free_running_drift(pb, torch, orc):
    """32 free-running timesteps (persistent kernel) against the oracle's own recurrence
    (literal Alg. 2 matvecs + double cell on its own h_t): the per-step parity bar holds
    at every step, so only rounding of the fp32 cell feeding later activation casts can
    separate the two; bound the drift of h and c over the run."""
    T, B, H, E, L = 32, 1, 512, 128, 4
    s = synth.seed(7, 4242)
    Wih, Whh = synth.weights(4 * H, E, s), synth.weights(4 * H, H, s + 1)
    bias = (synth.bias(4 * H, s + 2) + synth.bias(4 * H, s + 3)).astype(np.float32)
    x = np.stack([synth.activations(B, E, s + 10 + t, "gauss") for t in range(T)])
    h0, c0 = synth.activations(B, H, s + 4, "tanh"), synth.activations(B, H, s + 5, "gauss")
    Wih_i, Whh_i, bias_i = pb.interleave_gates(Wih), pb.interleave_gates(Whh), pb.interleave_gates(bias)
    wih, whh = pb.PackedWeights.quantize(Wih_i, L), pb.PackedWeights.quantize(Whh_i, L)
    ci, si, oi, _ = orc.quantize_weights(Wih_i, L, "grid")
    ch, sh, oh, _ = orc.quantize_weights(Whh_i, L, "grid")
    D = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    h_seq, c_last = pb.lstm_seq(D(x), D(h0), D(c0), wih, whh, D(bias_i))
    torch.cuda.synchronize()
    hs = h_seq.cpu().numpy()
    h_t, c_t = h0, c0
    worst = 0.0
    for t in range(T):
        _, yi, _ = orc.pbatch(ci, L, oi, si, L, x[t], 16)
        _, yh, _ = orc.pbatch(ch, L, oh, sh, L, h_t, 16)
        g = pb.deinterleave_gates((yi.astype(np.float64) + bias_i + yh.astype(np.float64)).T).T
        h_t, c_t = orc.lstm_cell(g, c_t)
        h_t = h_t.astype(np.float32)
        worst = max(worst, float(np.abs(hs[t] - h_t).max()))
    assert worst < 1e-3, worst
    assert float(np.abs(c_last.cpu().numpy() - c_t).max()) < 1e-3
