"""The NCCL row-shard entry point (pb_matmul_rowshard) on one GPU: a
single-rank communicator runs the same code path (local shard matvec,
in-place ncclAllGather for batch 1, gather + permute kernel for batch > 1),
and must give the oracle's y (acc-exact dequant, reading G13: identical bits)
and, bit-identically, pb_matmul's.  Multi-rank host logic is
covered on CPU by tests/test_shard_gloo.py."""
import ctypes as C

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


@pytest.mark.parametrize("R,K,L,B", [(4096, 2048, 4, 1), (1000, 784, 3, 3), (2048, 4096, 8, 2)])
def test_rowshard_single_rank_matches_oracle(pb, orc, R, K, L, B):
    import torch
    idb = (C.c_ubyte * 128)()
    st = pb.pb_comm_unique_id(C.cast(idb, C.c_void_p))
    if st == pb.PB_ENCCL:
        pytest.skip("NCCL not loadable: " + pb.pb_last_error().decode())
    pb.check(st)
    h = C.c_void_p()
    pb.check(pb.pb_comm_init(C.byref(h), C.cast(idb, C.c_void_p), 1, 0))
    try:
        m = synth.codes(R, K, L, 5)
        w = pb.PackedWeights.from_codes(pb.shard_codes(m, 1, 0), L, 0, 0.25)
        x = torch.from_numpy(synth.activations(B, K, 6)).cuda()
        y_ref = pb.matmul(x, w, L, 16)
        y = torch.full((B, R), np.nan, device="cuda")
        nb = pb.pb_rowshard_workspace_bytes(B, K, 16, R, 1)
        ws = pb.Workspace(nb)
        s = torch.cuda.current_stream().cuda_stream
        pb.check(pb.pb_matmul_rowshard(x.data_ptr(), B, C.byref(w.desc), R, L, 16, pb.PB_ACT_AUTO, y.data_ptr(),
                                       h, ws.ptr, ws.nbytes, s))
        torch.cuda.synchronize()
        _, y_o, _ = orc.pbatch(m, L, 0, 0.25, L, x.cpu().numpy(), 16, nthreads=8)
        assert np.array_equal(y.cpu().numpy().view(np.uint32), y_o.view(np.uint32))
        assert torch.equal(y.view(torch.int32), y_ref.view(torch.int32))
    finally:
        pb.pb_comm_destroy(h)
