"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
element by element on the same seeded inputs.

Bar (north star): integer accumulators bit-exact; dequantised y within
1e-5 relative (the G13 op sequence makes them bit-identical, also asserted).
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

RTOL = 1e-5


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


ENGINES = ["popc", "auto", "mma"]


def _engine(pb, name):
    return {"popc": pb.PB_ENGINE_POPC, "auto": pb.PB_ENGINE_AUTO, "mma": pb.PB_ENGINE_MMA}[name]


def run_gpu(pb, torch, codes, L, offset, scale, k_used, x, a, act_frac=-1024, engine="auto"):
    w = pb.PackedWeights.from_codes(codes, L, offset, scale)
    xd = torch.from_numpy(x).cuda()
    B = x.shape[0]
    acc = torch.full((B, codes.shape[0]), 0x5A5A5A5A, dtype=torch.int64, device="cuda")
    pb.set_engine(_engine(pb, engine))
    try:
        y = pb.matmul(xd, w, k_used, a, act_frac, acc=acc)
    finally:
        pb.set_engine(pb.PB_ENGINE_AUTO)
    torch.cuda.synchronize()
    return acc.cpu().numpy(), y.cpu().numpy()


def compare(acc, y, acc_o, y_o):
    assert np.array_equal(acc, acc_o), f"acc mismatch at {np.argwhere(acc != acc_o)[:5].tolist()}"
    np.testing.assert_allclose(y, y_o, rtol=RTOL, atol=0)
    assert np.array_equal(y.view(np.uint32), y_o.view(np.uint32))      # G13: identical bits


CASES = [  # R, K, B, L, k_used, a
    (1029, 784, 1, 4, 4, 16),     # C1 shape, ragged R
    (1024, 784, 1, 4, 2, 16),
    (10, 1000, 3, 8, 8, 8),
    (257, 4109, 2, 2, 2, 16),
    (33, 33, 16, 16, 16, 32),
    (100, 31, 128, 3, 3, 7),
    (1, 1, 1, 5, 5, 1),
    (3, 32, 2, 7, 1, 2),
    (65, 4109, 1, 12, 6, 31),
    (130, 129, 5, 16, 9, 3),
    (512, 2048, 16, 6, 6, 16),
    (300, 2000, 4, 8, 8, 16),     # N = 64 in one tensor-engine launch
    (257, 1030, 3, 5, 4, 16),     # N = 48 -> padded to 64
    (129, 3000, 8, 8, 7, 8),      # N = 64, a = 8
    (200, 1500, 37, 4, 4, 16),    # 10 slices of <= 4 columns, ragged last slice
    (512, 2048, 8, 16, 16, 16),   # 2 accumulator groups: N = 64 slices narrowed to N = 32
    # wide mode (a*B > 64, a >= 8): every 128-plane-column slice in one launch
    (300, 2000, 9, 8, 8, 16),     # 2 slices (8 + 1 columns), ragged K
    (1000, 4109, 40, 6, 5, 8),    # a = 8: 3 slices of 16/16/8, odd k_used
    (129, 3000, 24, 4, 4, 32),    # a = 32: 6 slices of 4
    (2048, 1024, 128, 2, 2, 16),  # 16 slices, 512 units over the grid
    (700, 5000, 19, 12, 11, 10),  # a = 10: slices of 12 columns (120 rows + 8 padding), 2 slices
    (257, 1030, 17, 1, 1, 16),    # L = 1 (canonical single layer) in wide mode
]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("R,K,B,L,k_used,a", CASES)
def test_parity_codes(pb, torch, orc, engine, R, K, B, L, k_used, a):
    s = synth.seed(2, R + 7 * K + 13 * B + L)
    m = synth.codes(R, K, L, s)
    x = synth.inject_edges(synth.activations(B, K, s + 1, "gauss"), s + 2)
    try:
        acc, y = run_gpu(pb, torch, m, L, 0, 0.0123, k_used, x, a, engine=engine)
    except pb.PBError as e:
        if engine == "mma" and e.status == pb.PB_EINVAL:
            pytest.skip("mma engine does not cover this shape")
        raise
    acc_o, y_o, _ = orc.pbatch(m, L, 0, 0.0123, k_used, x, a, nthreads=8)
    compare(acc, y, acc_o, y_o)


@pytest.mark.parametrize("R,K,B", [(64, 32, 5), (1000, 784, 1), (7, 3000, 3)])
def test_parity_binary(pb, torch, orc, R, K, B):
    s = synth.seed(2, 500 + R)
    m = synth.binary_codes(R, K, s)
    x = synth.activations(B, K, s + 1, "relu")
    acc, y = run_gpu(pb, torch, m, 1, 1, 0.37, 1, x, 16)
    acc_o, y_o, _ = orc.pbatch(m, 1, 1, 0.37, 1, x, 16)
    compare(acc, y, acc_o, y_o)


@pytest.mark.parametrize("L", list(range(1, 17)))
def test_parity_every_L_every_kused(pb, torch, orc, L):
    R, K, B, a = 77, 300, 2, 16
    s = synth.seed(2, 900 + L)
    if L == 1:
        m, off = synth.binary_codes(R, K, s), 1
    else:
        m, off = synth.codes(R, K, L, s), 0
    x = synth.activations(B, K, s + 1, "tanh")
    w = pb.PackedWeights.from_codes(m, L, off, 1.0)
    xd = torch.from_numpy(x).cuda()
    for k in range(1, L + 1):
        acc = torch.zeros((B, R), dtype=torch.int64, device="cuda")
        y = pb.matmul(xd, w, k, a, acc=acc)
        acc_o, y_o, _ = orc.pbatch(m, L, off, 1.0, k, x, a)
        compare(acc.cpu().numpy(), y.cpu().numpy(), acc_o, y_o)


def test_parity_literal_alg2_cast(pb, torch, orc):
    # act_frac = 16 with a = 32 is exactly Alg. 2 line 1, saturating
    R, K, B, L = 50, 500, 3, 8
    m = synth.codes(R, K, L, 7)
    x = synth.activations(B, K, 8, "gauss")
    x[0, 0] = 1e6       # saturates at 2^31 - 1
    for a, frac in [(32, 16), (16, 8), (8, 0)]:
        acc, y = run_gpu(pb, torch, m, L, 0, 1.0, L, x, a, act_frac=frac)
        acc_o, y_o, _ = orc.pbatch(m, L, 0, 1.0, L, x, a, act_frac=frac)
        compare(acc, y, acc_o, y_o)


def test_parity_quantizer_path(pb, torch, orc):
    # float W through the library packer vs oracle quantiser, all modes
    R, K, B = 300, 1000, 2
    W = synth.weights(R, K, 11, "student_t")
    x = synth.activations(B, K, 12, "mnist")
    xd = torch.from_numpy(x).cuda()
    for mode, L, name in [(pb.PB_Q_GRID, 4, "grid"), (pb.PB_Q_ALG1, 6, "alg1"), (pb.PB_Q_BINARY, 1, "binary"),
                          (pb.PB_Q_GRID, 16, "grid")]:
        w = pb.PackedWeights.quantize(W, L, mode)
        codes, s, off, _ = orc.quantize_weights(W, L, name)
        assert w.scale == s and w.offset == off
        acc = torch.zeros((B, R), dtype=torch.int64, device="cuda")
        y = pb.matmul(xd, w, L, 16, acc=acc)
        acc_o, y_o, _ = orc.pbatch(codes, L, off, s, L, x, 16)
        compare(acc.cpu().numpy(), y.cpu().numpy(), acc_o, y_o)


def test_edge_cases(pb, torch, orc):
    # all-zero x, subnormal column maximum, negative powers of two, K = 1
    R, K, L = 40, 64, 5
    m = synth.codes(R, K, L, 3)
    x = np.zeros((4, K), np.float32)
    x[1, :] = np.float32(1e-41)
    x[1, 5] = np.float32(-3e-41)
    x[2, :] = -np.float32(2.0) ** -(np.arange(K, dtype=np.float32) % 7)
    x[3, ::3] = np.float32(-0.5)
    acc, y = run_gpu(pb, torch, m, L, 0, 0.25, L, x, 16)
    acc_o, y_o, f = orc.pbatch(m, L, 0, 0.25, L, x, 16)
    compare(acc, y, acc_o, y_o)
    assert not acc[0].any() and f[0] == 0
    m1 = synth.codes(9, 1, 3, 4)
    x1 = synth.activations(2, 1, 5)
    acc, y = run_gpu(pb, torch, m1, 3, 0, 1.0, 3, x1, 8)
    acc_o, y_o, _ = orc.pbatch(m1, 3, 0, 1.0, 3, x1, 8)
    compare(acc, y, acc_o, y_o)


def test_empty_shapes(pb, torch):
    w = pb.PackedWeights.from_codes(np.zeros((0, 64), np.int32), 4)
    y = pb.matmul(torch.zeros((2, 64), device="cuda"), w, 4, 16)
    assert y.shape == (2, 0)
    w = pb.PackedWeights.from_codes(np.zeros((8, 64), np.int32), 4)
    y = pb.matmul(torch.zeros((0, 64), device="cuda"), w, 4, 16)
    assert y.shape == (0, 8)


def test_latency_drops_with_fewer_layers(pb, torch):
    # north star: latency drops with fewer weight bitlayers (ordering only)
    R = K = 8192
    m = synth.codes(R, K, 16, 99)
    w = pb.PackedWeights.from_codes(m, 16)
    x = torch.randn(1, K, device="cuda")
    ws = pb.Workspace(pb.workspace_bytes(1, K, 16))
    y = torch.empty(1, R, device="cuda")
    times = {}
    for k in (16, 8, 4, 2, 1):
        for _ in range(3):
            pb.matmul(x, w, k, 16, y=y, ws=ws)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20):
            pb.matmul(x, w, k, 16, y=y, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        times[k] = e0.elapsed_time(e1) / 20
    assert times[16] > times[8] > times[4] > times[1], times


@pytest.mark.parametrize("R,K,B,L,k_used,a", [(1024, 8192, 1, 4, 4, 16), (1000, 3000, 2, 8, 5, 16),
                                              (300, 4096, 4, 3, 3, 8), (129, 1000, 1, 16, 16, 16),
                                              (2048, 2048, 1, 8, 8, 32), (640, 6000, 3, 2, 2, 5),
                                              # many units per CTA (dynamic claims), two accumulator
                                              # groups (L=16, K=8192: 5 passes per group), batch columns
                                              (4096, 8192, 1, 8, 8, 16), (4000, 8192, 1, 16, 11, 16),
                                              (8192, 8192, 1, 4, 4, 16), (4096, 8100, 3, 6, 5, 8)])
def test_tc_streamk_repeat(pb, torch, orc, R, K, B, L, k_used, a):
    # tensor engine: stream-K partial tiles + self-cleaning scratch across calls
    s = synth.seed(2, 3000 + R + K)
    m = synth.codes(R, K, L, s)
    x = synth.inject_edges(synth.activations(B, K, s + 1, "gauss"), s + 2)
    w = pb.PackedWeights.from_codes(m, L, 0, 0.5)
    ws = pb.Workspace(pb.workspace_bytes(B, K, a))
    xd = torch.from_numpy(x).cuda()
    acc_o, y_o, _ = orc.pbatch(m, L, 0, 0.5, k_used, x, a, nthreads=8)
    pb.set_engine(pb.PB_ENGINE_MMA)
    try:
        for rep in range(3):
            acc = torch.zeros((B, R), dtype=torch.int64, device="cuda")
            y = pb.matmul(xd, w, k_used, a, acc=acc, ws=ws)
            torch.cuda.synchronize()
            compare(acc.cpu().numpy(), y.cpu().numpy(), acc_o, y_o)
    finally:
        pb.set_engine(pb.PB_ENGINE_AUTO)


@pytest.mark.parametrize("engine", ["popc", "auto"])
@pytest.mark.parametrize("R,K,B,L,k_used,a", [(1029, 784, 1, 4, 2, 16), (300, 4109, 3, 8, 5, 16),
                                              (4096, 8192, 1, 8, 3, 16), (129, 1000, 2, 16, 9, 8),
                                              (257, 1030, 1, 6, 6, 16)])
def test_parity_midpoint(pb, torch, orc, engine, R, K, B, L, k_used, a):
    # pb_matmul_ex(PB_MM_MIDPOINT) against the oracle's midpoint option
    s = synth.seed(2, 7000 + R + K + L)
    m = synth.codes(R, K, L, s)
    x = synth.inject_edges(synth.activations(B, K, s + 1, "gauss"), s + 2)
    w = pb.PackedWeights.from_codes(m, L, 0, 0.0123)
    xd = torch.from_numpy(x).cuda()
    acc = torch.zeros((B, R), dtype=torch.int64, device="cuda")
    pb.set_engine(_engine(pb, engine))
    try:
        y = pb.matmul(xd, w, k_used, a, acc=acc, midpoint=True)
    finally:
        pb.set_engine(pb.PB_ENGINE_AUTO)
    torch.cuda.synchronize()
    acc_o, y_o, _ = orc.pbatch(m, L, 0, 0.0123, k_used, x, a, nthreads=8, midpoint=True)
    compare(acc.cpu().numpy(), y.cpu().numpy(), acc_o, y_o)
