"""Exactness of the tensor engine's f32 TMEM accumulator at its bound.

The tensor engine sums the 0/1 products of one accumulator group (G layers,
reading G10: exact integers) in an f32 TMEM accumulator, which is exact while
every partial sum is an integer < 2^24; make_plan (pb_gemm_tc.cu) sizes the
groups so that K_pad * (2^G - 1) <= 2^24.  Random inputs never get near that:
here every product is at its maximum.

  * codes m = 2^(L-1) - 1 everywhere: the (complemented) sign layer and every
    magnitude layer hold 1 in every column, so every A nibble is 0b11;
  * x = -2^-16 with the literal Alg. 2 cast act_frac = 16: x_q = -1,
    i.e. every one of the a activation planes is all ones.

So every group sum sits at K * (2^G - 1), and the closed form of the result is
acc = sum_c m * x_q = -K (2^(L-1) - 1) for every row and batch column --
checked against that closed form (independent of the oracle) and against the
oracle's literal Alg. 2.  Shapes: K = 16384 with L = 8 (one group), L = 10 (one
group of 5 passes: 16384 * 1023 = 16,760,832, just under 2^24) and L = 16 (two
groups), and the G thresholds at K = 4096 (G = 12: 4096 * 4095) and K = 4097
(the next K pads to 4224 columns, G drops to 11), K = 65536 (G = 8)."""
import numpy as np
import pytest

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


@pytest.mark.parametrize("R,K,L,B", [(128, 16384, 8, 1), (130, 16384, 10, 1), (256, 16384, 16, 1),
                                     (128, 4096, 12, 1), (129, 4097, 12, 1), (128, 4096, 12, 4),
                                     (128, 65536, 8, 1), (200, 16384, 16, 2)])
def test_all_max_products(pb, torch, orc, R, K, L, B):
    a, act_frac = 16, 16
    codes = np.full((R, K), (1 << (L - 1)) - 1, dtype=np.int32)
    x = np.full((B, K), -2.0 ** -16, dtype=np.float32)
    w = pb.PackedWeights.from_codes(codes, L, 0, 0.5)
    acc = torch.zeros((B, R), dtype=torch.int64, device="cuda")
    for engine in (pb.PB_ENGINE_MMA, pb.PB_ENGINE_AUTO):
        pb.set_engine(engine)
        try:
            y = pb.matmul(torch.from_numpy(x).cuda(), w, L, a, act_frac, acc=acc)
        finally:
            pb.set_engine(pb.PB_ENGINE_AUTO)
        torch.cuda.synchronize()
        acc_g = acc.cpu().numpy()
        closed = -K * ((1 << (L - 1)) - 1)
        assert (acc_g == closed).all(), (engine, np.unique(acc_g)[:4], closed)
        acc_o, y_o, _ = orc.pbatch(codes, L, 0, 0.5, L, x, a, act_frac=act_frac, nthreads=8)
        assert np.array_equal(acc_g, acc_o)
        assert np.array_equal(y.cpu().numpy().view(np.uint32), y_o.view(np.uint32))


@pytest.mark.parametrize("L,k_used", [(16, 11), (16, 1), (9, 9)])
def test_all_max_products_truncated(pb, torch, orc, L, k_used):
    # k_used < L floor-truncates the codes (reading G12): m_trunc = 2^(L-1) - 2^(L-k_used)
    R, K, a = 128, 16384, 16
    codes = np.full((R, K), (1 << (L - 1)) - 1, dtype=np.int32)
    x = np.full((1, K), -2.0 ** -16, dtype=np.float32)
    w = pb.PackedWeights.from_codes(codes, L, 0, 1.0)
    acc = torch.zeros((1, R), dtype=torch.int64, device="cuda")
    pb.matmul(torch.from_numpy(x).cuda(), w, k_used, a, 16, acc=acc)
    torch.cuda.synchronize()
    m_trunc = (1 << (L - 1)) - (1 << (L - k_used))
    assert (acc.cpu().numpy() == -K * m_trunc).all()
    acc_o, _, _ = orc.pbatch(codes, L, 0, 1.0, k_used, x, a, act_frac=16, nthreads=8)
    assert np.array_equal(acc.cpu().numpy(), acc_o)
