"""Exactness of the tensor engine's f32 TMEM accumulator at its bound.

The tensor engine sums the products of one accumulator group (G layers, reading
G10: exact integers) in an f32 TMEM accumulator, which is exact while every
partial sum is an integer of magnitude < 2^24.  Per pass and column the product
is (2 W_hi + W_lo) * d with the activation digit d = 2 X_2k + X_2k+1 in [-2, 3]
(pb_common.cuh), so make_plan sizes the groups with 3 K_pad 2^G <= 2^24.
Random inputs never get near that; here every product is at its maximum.

  * codes m = 2^(L-1) - 1 everywhere: the (complemented) sign layer and every
    magnitude layer hold 1 in every column, so every A nibble is 0b11 (1.5);
  * with the literal Alg. 2 cast act_frac = 16: x = (2^15 - 1) 2^-16
    gives x_q = 2^15 - 1, every digit 3 (the maximum product 9); x = -2^-16
    gives x_q = -1, every plane 1 (the sign digit -1, the others 3).

The closed form of the result is acc = sum_c m x_q = K (2^(L-1) - 1) x_q for
every row and batch column -- checked against that closed form (independent of
the oracle) and against the oracle's literal Alg. 2.  Shapes: K = 16384 with
L = 8 (one group of 4 passes: 16384 * 9 * 85), L = 10 and 16 (two groups);
K = 5376, the largest padded K with G = 10, at L = 10 (one group of 5 passes:
5376 * 9 * 341 = 16,498,944, just under 2^24) and K = 5377 (pads to 5504: G
drops to 9); K = 4096 / 4097 at L = 12 and K = 65536 (G = 6)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

XQ = {"pos": ((1 << 15) - 1) * 2.0 ** -16, "neg": -2.0 ** -16}


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


@pytest.mark.parametrize("sign", ["pos", "neg"])
@pytest.mark.parametrize("R,K,L,B", [(128, 16384, 8, 1), (130, 16384, 10, 1), (256, 16384, 16, 1),
                                     (128, 5376, 10, 1), (129, 5377, 10, 3), (128, 4096, 12, 1),
                                     (129, 4097, 12, 1), (128, 4096, 12, 4), (128, 65536, 8, 1),
                                     (200, 16384, 16, 2), (256, 5376, 10, 20)])
def test_all_max_products(pb, torch, orc, R, K, L, B, sign):
    a, act_frac = 16, 16
    codes = np.full((R, K), (1 << (L - 1)) - 1, dtype=np.int32)
    x = np.full((B, K), XQ[sign], dtype=np.float32)
    xq = round(XQ[sign] * 2 ** 16)
    w = pb.PackedWeights.from_codes(codes, L, 0, 0.5)
    acc = torch.zeros((B, R), dtype=torch.int64, device="cuda")
    acc_o, y_o, _ = orc.pbatch(codes, L, 0, 0.5, L, x, a, act_frac=act_frac, nthreads=8)
    closed = K * ((1 << (L - 1)) - 1) * xq
    assert (acc_o == closed).all()
    for engine in (pb.PB_ENGINE_MMA, pb.PB_ENGINE_AUTO):
        pb.set_engine(engine)
        try:
            y = pb.matmul(torch.from_numpy(x).cuda(), w, L, a, act_frac, acc=acc)
        except pb.PBError as e:
            if engine == pb.PB_ENGINE_MMA and e.status == pb.PB_EINVAL:
                continue             # the tensor engine does not take this shape in one launch
            raise
        finally:
            pb.set_engine(pb.PB_ENGINE_AUTO)
        torch.cuda.synchronize()
        acc_g = acc.cpu().numpy()
        assert (acc_g == closed).all(), (engine, np.unique(acc_g)[:4], closed)
        assert np.array_equal(acc_g, acc_o)
        assert np.array_equal(y.cpu().numpy().view(np.uint32), y_o.view(np.uint32))


@pytest.mark.parametrize("L,k_used", [(16, 11), (16, 1), (9, 9), (10, 7)])
def test_all_max_products_truncated(pb, torch, orc, L, k_used):
    # k_used < L floor-truncates the codes (reading G12): m_trunc = 2^(L-1) - 2^(L-k_used)
    R, K, a = 128, 16384, 16
    codes = np.full((R, K), (1 << (L - 1)) - 1, dtype=np.int32)
    x = np.full((1, K), XQ["pos"], dtype=np.float32)
    w = pb.PackedWeights.from_codes(codes, L, 0, 1.0)
    acc = torch.zeros((1, R), dtype=torch.int64, device="cuda")
    pb.matmul(torch.from_numpy(x).cuda(), w, k_used, a, 16, acc=acc)
    torch.cuda.synchronize()
    m_trunc = (1 << (L - 1)) - (1 << (L - k_used))
    assert (acc.cpu().numpy() == K * m_trunc * ((1 << 15) - 1)).all()
    acc_o, _, _ = orc.pbatch(codes, L, 0, 1.0, k_used, x, a, act_frac=16, nthreads=8)
    assert np.array_equal(acc.cpu().numpy(), acc_o)
