"""CPU tests of the C-ABI library: it loads, exports every symbol that
include/pb.h declares, and its host-side logic (offline packer, validation,
row sharding, memory model) agrees with the oracle / the paper.  No compute
call reaches the GPU here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import synth
from packed_layout import unpack_layers, unpack_layers_full

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pb():
    import build_pb
    build_pb.build()
    import paper_2003_00822_b200 as pb
    return pb


def _declared():
    src = open(os.path.join(ROOT, "include", "pb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pb_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(pb):
    names = _declared()
    assert len(names) >= 20
    lib = C.CDLL(pb.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(pb.EXPORTED)
    assert b"sm_100a" in pb.pb_version()


def test_library_is_sm100a_cubin(pb):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pb.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _host_pack(pb, W, L, mode, clip=0.0):
    R, K = W.shape
    buf = np.zeros(max(1, pb.pb_packed_bytes(R, K, L) // 4), np.uint32)
    d = pb.pb_weights()
    st = pb.pb_quantize_pack_weights(W.ctypes.data, R, K, L, mode, clip, buf.ctypes.data, 0, None, C.byref(d))
    return st, d, buf


def _unpack(buf, L, R, K):
    return unpack_layers(buf, L, R, K)


@pytest.mark.parametrize("R,K,L,mode", [(5, 37, 4, "grid"), (3, 128, 2, "grid"), (7, 300, 8, "grid"),
                                        (4, 129, 16, "grid"), (6, 33, 3, "alg1"), (5, 200, 8, "alg1"),
                                        (9, 31, 1, "binary"), (2, 1, 5, "grid")])
def test_packer_matches_oracle_decomposition(pb, orc, R, K, L, mode):
    W = synth.weights(R, K, synth.seed(1, R * 7 + K), "student_t")
    m = {"grid": pb.PB_Q_GRID, "alg1": pb.PB_Q_ALG1, "binary": pb.PB_Q_BINARY}[mode]
    st, d, buf = _host_pack(pb, W, L, m)
    assert st == pb.PB_OK, pb.pb_last_error()
    codes, s, off, ost = orc.quantize_weights(W, L, mode)
    assert d.scale == s and d.offset == off and d.layers == L and d.kwords == 4 * ((K + 127) // 128)
    bits = _unpack(buf, L, R, K)
    if mode == "binary":
        ref = (codes == -1).astype(np.uint8)[None]
    else:
        ref = orc.decompose(codes, L)
    assert np.array_equal(bits, ref)
    # padding columns are zero (AND-neutral)
    kw = 4 * ((K + 127) // 128)
    assert not unpack_layers_full(buf, L, R, K)[:, :, K:].any()


def test_packer_clip_and_degenerate(pb, orc):
    W = synth.weights(6, 64, 3, "student_t")
    st, d, buf = _host_pack(pb, W, 5, pb.PB_Q_GRID, clip=0.05)
    codes, s, _, _ = orc.quantize_weights(W, 5, "grid", clip=float(np.float32(0.05)))  # the ABI takes a float clip
    assert st == pb.PB_OK and d.scale == s
    assert np.array_equal(_unpack(buf, 5, 6, 64), orc.decompose(codes, 5))
    Z = np.zeros((3, 40), np.float32)
    st, d, buf = _host_pack(pb, Z, 4, pb.PB_Q_GRID)
    assert st == pb.PB_EDEGENERATE and d.scale == 1.0 and not buf.any()


@pytest.mark.parametrize("L", [2, 3, 8, 16])
def test_grid_step_matches_oracle(pb, orc, L):
    # pb_grid_step from a layer's extrema == the oracle quantiser's d on the whole layer,
    # also when the extrema are all-reduced over row shards (the max/min of the shards' extrema)
    W = synth.weights(37, 300, synth.seed(1, L), "student_t")
    _, d_or, _ = orc.quantize_round(W, L - 1)
    shards = np.array_split(W, 3)
    mn = min(float(s.min()) for s in shards)
    mx = max(float(s.max()) for s in shards)
    assert pb.grid_step(mn, mx, L) == d_or
    # reading G5: constant W -> |c| (PB_EDEGENERATE), all-zero -> 1; bad arguments
    d = C.c_double()
    assert pb.pb_grid_step(-0.25, -0.25, L, C.byref(d)) == pb.PB_EDEGENERATE and d.value == 0.25
    assert orc.quantize_round(np.full((2, 3), -0.25, np.float32), L - 1)[1] == 0.25
    assert pb.pb_grid_step(0.0, 0.0, L, C.byref(d)) == pb.PB_EDEGENERATE and d.value == 1.0
    assert pb.pb_grid_step(1.0, 0.0, L, C.byref(d)) == pb.PB_EINVAL
    assert pb.pb_grid_step(0.0, 1.0, 1, C.byref(d)) == pb.PB_EINVAL
    assert pb.pb_grid_step(0.0, float("inf"), L, C.byref(d)) == pb.PB_EINVAL


def test_pack_codes_and_range(pb, orc):
    m = synth.codes(4, 77, 6, 9)
    buf = np.zeros(pb.pb_packed_bytes(4, 77, 6) // 4, np.uint32)
    d = pb.pb_weights()
    assert pb.pb_pack_codes(m.ctypes.data, 4, 77, 6, 0, 0.5, buf.ctypes.data, 0, None, C.byref(d)) == pb.PB_OK
    assert np.array_equal(_unpack(buf, 6, 4, 77), orc.decompose(m, 6))
    bad = m.copy()
    bad[0, 0] = 32
    assert pb.pb_pack_codes(bad.ctypes.data, 4, 77, 6, 0, 0.5, buf.ctypes.data, 0, None, C.byref(d)) == pb.PB_ERANGE


def test_search_clip_matches_oracle(pb, orc):
    W = np.concatenate([np.random.default_rng(5).uniform(-0.1, 0.1, 4999), [1.0]]).astype(np.float32)
    t = C.c_float()
    assert pb.pb_search_clip(W.ctypes.data, 1, W.size, 5, C.byref(t)) == pb.PB_OK
    t_or, _ = orc.search_clip(W, 5)
    assert t.value == t_or


def test_memory_model(pb):
    # P:124 / P:249: packed bytes = L*R*K/8 when K % 128 == 0; ratio vs fp32 = 32/L
    for L in range(1, 17):
        assert pb.pb_packed_bytes(1024, 1024, L) == L * 1024 * 1024 // 8
        assert 4 * 1024 * 1024 / pb.pb_packed_bytes(1024, 1024, L) == pytest.approx(32 / L)
    assert pb.pb_kwords(1) == 4 and pb.pb_kwords(128) == 4 and pb.pb_kwords(129) == 8 and pb.pb_kwords(0) == 0


def test_validation_before_launch(pb):
    # every argument error is reported before any CUDA call (no device here)
    d = pb.pb_weights(16, 8, 64, 4, 4, 0, 1.0)
    wsn = pb.pb_workspace_bytes(1, 64, 16)
    # dominated by the partial-tile sums: 2048 tiles x min(32, 64/ceil(a/2)) batch columns x 128 x 8 B
    # (activation digits: 2 planes per MMA column; 16 MiB at a=16)
    assert wsn <= 17 << 20
    ws = np.zeros(wsn + 256, np.uint8)
    wsp = (ws.ctypes.data + 255) // 256 * 256
    y = np.zeros(64, np.float32)
    args = lambda k, a, frac=pb.PB_ACT_AUTO: (16, 1, C.byref(d), k, a, frac, y.ctypes.data, None, wsp, wsn, None)
    assert pb.pb_matmul(*args(0, 16)) == pb.PB_EINVAL
    assert pb.pb_matmul(*args(5, 16)) == pb.PB_EINVAL
    assert b"k_used" in pb.pb_last_error()
    assert pb.pb_matmul(*args(4, 0)) == pb.PB_EINVAL
    assert pb.pb_matmul(*args(4, 33)) == pb.PB_EINVAL
    assert pb.pb_matmul(*args(4, 16, 500)) == pb.PB_EINVAL
    small = (16, 1, C.byref(d), 4, 16, pb.PB_ACT_AUTO, y.ctypes.data, None, wsp, 8, None)
    assert pb.pb_matmul(*small) == pb.PB_EINVAL and b"workspace" in pb.pb_last_error()
    # reading G11 overflow guard: L=16, a=32 allows K <= 2^14 ... 2^16? bound = log2K + 46 <= 62
    big = pb.pb_weights(16, 1, 1 << 17, 4 * ((1 << 17) // 128), 16, 0, 1.0)
    wsb = np.zeros(pb.pb_workspace_bytes(1, 1 << 17, 32) + 256, np.uint8)
    wbp = (wsb.ctypes.data + 255) // 256 * 256
    assert pb.pb_matmul(16, 1, C.byref(big), 16, 32, pb.PB_ACT_AUTO, y.ctypes.data, None, wbp,
                        pb.pb_workspace_bytes(1, 1 << 17, 32), None) == pb.PB_ERANGE
    bad_off = pb.pb_weights(16, 8, 64, 4, 4, 1, 1.0)
    assert pb.pb_matmul(16, 1, C.byref(bad_off), 1, 16, pb.PB_ACT_AUTO, y.ctypes.data, None, wsp, wsn,
                        None) == pb.PB_EINVAL
    mis = pb.pb_weights(20, 8, 64, 4, 4, 0, 1.0)   # misaligned bits
    assert pb.pb_matmul(*(16, 1, C.byref(mis), 4, 16, pb.PB_ACT_AUTO, y.ctypes.data, None, wsp, wsn,
                          None)) == pb.PB_EINVAL
    assert pb.pb_set_engine(7) == pb.PB_EINVAL


@pytest.mark.parametrize("R,N", [(16384, 8), (10, 3), (7, 8), (1024, 1), (5, 2)])
def test_shard_rows_partition(pb, R, N):
    seen = []
    rs = (R + N - 1) // N
    for g in range(N):
        r0, n = pb.shard_rows(R, N, g)
        assert 0 <= n <= rs
        seen.extend(range(r0, r0 + n))
    assert seen == list(range(R))


def test_workspace_layout(pb):
    assert pb.pb_workspace_bytes(1, 16384, 16) >= 16 * 16384 // 8 + 16 * 16384
    assert pb.pb_workspace_bytes(128, 4096, 16) >= 128 * 16 * 4096 // 8
    assert pb.pb_workspace_bytes(1, 10, 0) == 0
    assert pb.pb_rowshard_workspace_bytes(4, 1024, 16, 1000, 8) >= pb.pb_workspace_bytes(4, 1024, 16) + 4 * 4 * 125 * 9


def test_p2p_argument_validation(pb):
    # the fused peer all-gather's setup rejects bad arguments before any CUDA call
    h = C.c_void_p()
    hb = C.create_string_buffer(int(pb.pb_p2p_handle_bytes()) or 64)
    assert pb.pb_p2p_create(C.byref(h), 3, 0, 1, 1024, hb) == pb.PB_EINVAL      # not 1, 2, 4 or 8 ranks
    assert pb.pb_p2p_create(C.byref(h), 2, 2, 1, 1024, hb) == pb.PB_EINVAL      # rank out of range
    assert pb.pb_p2p_create(C.byref(h), 16, 0, 1, 1024, hb) == pb.PB_EINVAL     # more than one node
    assert pb.pb_p2p_create(C.byref(h), 2, 0, 0, 1024, hb) == pb.PB_EINVAL      # empty batch
    assert pb.pb_p2p_open(None, hb) == pb.PB_EINVAL
    assert pb.pb_matmul_rowshard_p2p(None, 1, None, 1024, 1, 16, pb.PB_ACT_AUTO, None, None, 0, None) == pb.PB_EINVAL
    assert pb.pb_p2p_destroy(None) == pb.PB_OK
