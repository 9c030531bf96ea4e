"""GPU packer (pb_quantize_pack_weights_device): byte-identical
to the host packer (itself pinned to the oracle's decomposition in
tests/test_abi_host.py and the parity suites) for the PB_Q_GRID quantiser,
clipped grids, explicit (shard) grid steps and the degenerate cases of reading G5."""
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


def same(pb, a, b):
    assert a.status == b.status
    assert a.desc.scale == b.desc.scale and a.desc.offset == b.desc.offset
    assert (a.desc.rows, a.desc.cols, a.desc.kwords, a.desc.layers) == (b.desc.rows, b.desc.cols, b.desc.kwords,
                                                                        b.desc.layers)
    assert np.array_equal(a.buf.cpu().numpy(), b.buf.cpu().numpy())


@pytest.mark.parametrize("R,K", [(1, 1), (3, 31), (257, 1000), (1029, 784), (64, 4109)])
@pytest.mark.parametrize("L", [2, 3, 4, 7, 8, 13, 16])
def test_device_pack_matches_host(pb, torch, R, K, L):
    W = synth.weights(R, K, synth.seed(8, R + K + L))
    same(pb, pb.PackedWeights.quantize_device(torch.from_numpy(W).cuda(), L), pb.PackedWeights.quantize(W, L))


@pytest.mark.parametrize("L", [2, 5, 8])
def test_device_pack_clip_and_step(pb, torch, L):
    W = synth.weights(300, 2000, synth.seed(8, 77), "student_t")
    Wd = torch.from_numpy(W).cuda()
    t = float(np.abs(W).max() * 0.4)
    same(pb, pb.PackedWeights.quantize_device(Wd, L, clip=t), pb.PackedWeights.quantize(W, L, clip=t))
    step = 0.0123
    same(pb, pb.PackedWeights.quantize_device(Wd, L, step=step), pb.PackedWeights.quantize_step(W, L, step))


def test_device_pack_degenerate(pb, torch):
    for W in (np.zeros((5, 70), np.float32), np.full((5, 70), -0.25, np.float32)):
        a = pb.PackedWeights.quantize_device(torch.from_numpy(W).cuda(), 4)
        b = pb.PackedWeights.quantize(W, 4)
        assert a.status == pb.PB_EDEGENERATE
        same(pb, a, b)


def test_device_pack_full_size(pb, torch):
    # C5-sized pack (16384 x 16384, 1 GiB of fp32 W) on the GPU equals the host pack
    R = K = 16384
    W = synth.weights_rows(R, K, synth.seed(5, 0), 0, R)
    a = pb.PackedWeights.quantize_device(torch.from_numpy(W).cuda(), 8)
    b = pb.PackedWeights.quantize(W, 8)
    same(pb, a, b)
