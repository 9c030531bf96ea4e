"""Host-side logic of the row-sharded path with two processes
on the gloo backend (CPU): row partition + padding, the global Q(W) grid step
from all-reduced extrema (pb_quantize_pack_weights_step), the all-gather of
y shards and the [N][B][R/N] -> [B][R] permute.  Shard results come from the
oracle (no GPU here); the library's packer runs on the host."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, R, K, L, B, a, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import paper_2003_00822_b200 as pb
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W = synth.weights_rows(R, K, 77)            # every rank can draw any rows
        x = synth.activations(B, K, 78, "gauss")
        rs = (R + world - 1) // world
        r0, nr = pb.shard_rows(R, world, rank)
        Wl = np.zeros((rs, K), np.float32)
        Wl[:nr] = W[r0:r0 + nr]
        mn = torch.tensor([float(Wl[:nr].min()) if nr else np.inf], dtype=torch.float64)
        mx = torch.tensor([float(Wl[:nr].max()) if nr else -np.inf], dtype=torch.float64)
        dist.all_reduce(mn, dist.ReduceOp.MIN)
        dist.all_reduce(mx, dist.ReduceOp.MAX)
        step = pb.grid_step(mn.item(), mx.item(), L)
        # host pack of the shard with the global step
        buf = np.zeros(pb.pb_packed_bytes(rs, K, L) // 4, np.uint32)
        d = pb.pb_weights()
        assert pb.pb_quantize_pack_weights_step(Wl.ctypes.data, rs, K, L, step, buf.ctypes.data, 0, None,
                                                C.byref(d)) == pb.PB_OK
        # the unsharded layer's quantiser gives the same step and codes
        codes_full, s_full, _, _ = oracle.quantize_weights(W, L, "grid")
        assert step == s_full and d.scale == s_full
        kw = d.kwords
        from packed_layout import unpack_layers
        bits = unpack_layers(buf, L, rs, K, kw)[:, :nr]
        assert np.array_equal(bits, oracle.decompose(codes_full[r0:r0 + nr], L))
        # shard result (oracle stands in for the GPU), padded to rs rows, gathered
        codes_sh = np.zeros((rs, K), np.int32)
        codes_sh[:nr] = codes_full[r0:r0 + nr]
        _, y_sh, _ = oracle.pbatch(codes_sh, L, 0, step, L, x, a)           # [B][rs]
        gathered = [torch.zeros(B, rs) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(y_sh))
        g = torch.stack(gathered).numpy()                                   # [N][B][rs]
        y_full = g.transpose(1, 0, 2).reshape(B, world * rs)[:, :R]         # permute, drop padding
        _, y_ref, _ = oracle.pbatch(codes_full, L, 0, s_full, L, x, a)
        q.put((rank, bool(np.array_equal(y_full.view(np.uint32), y_ref.view(np.uint32)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("R,K,L,B", [(10, 70, 4, 1), (37, 130, 3, 3), (64, 64, 8, 2)])
def test_rowshard_two_ranks(R, K, L, B):
    import build_pb
    build_pb.build()
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, R, K, L, B, 16, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: True, 1: True}
