"""paper_2003_00822_b200 -- B200-native PrecisionBatching bitlayer matvec.

Thin Python binding over the C ABI of ``libpb.so`` (``include/pb.h``).  The
functions ``pb_*`` below have the same names and arguments as the C entry
points (argument marshalling only); every step of the hot path runs in the
library's sm_100a kernels.  Torch is used only for device memory and streams
in the convenience helpers (``PackedWeights``, ``matmul``, ...).

There is no CPU fallback: importing the package fails loudly when
``libpb.so`` has not been built (``python -m paper_2003_00822_b200.build``),
and compute calls fail with PB_ECUDA when no GPU is usable.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpb.so")

PB_OK, PB_EINVAL, PB_ERANGE, PB_EDEGENERATE, PB_ECUDA, PB_ENCCL = range(6)
PB_Q_GRID, PB_Q_ALG1, PB_Q_BINARY = 0, 1, 2
PB_ACT_AUTO = -1024
PB_FN_NONE, PB_FN_RELU, PB_FN_TANH, PB_FN_SIGMOID = 0, 1, 2, 3
PB_ENGINE_AUTO, PB_ENGINE_POPC, PB_ENGINE_MMA = 0, 1, 2
_STATUS = {0: "PB_OK", 1: "PB_EINVAL", 2: "PB_ERANGE", 3: "PB_EDEGENERATE", 4: "PB_ECUDA", 5: "PB_ENCCL"}

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python build_pb.py` "
                      "(there is no CPU fallback)")


class pb_weights(C.Structure):
    _fields_ = [("bits", C.c_void_p), ("rows", C.c_int64), ("cols", C.c_int64), ("kwords", C.c_int64),
                ("layers", C.c_int32), ("offset", C.c_int32), ("scale", C.c_double)]


_lib = C.CDLL(LIB_PATH)
_p, _i64, _i32, _sz, _dbl, _f32 = C.c_void_p, C.c_int64, C.c_int32, C.c_size_t, C.c_double, C.c_float
_W = C.POINTER(pb_weights)

_SIGS = {
    "pb_last_error": ([], C.c_char_p),
    "pb_version": ([], C.c_char_p),
    "pb_debug_timeline": ([_p, _i64], _i64),
    "pb_kwords": ([_i64], _i64),
    "pb_packed_bytes": ([_i64, _i64, _i32], _sz),
    "pb_quantize_pack_weights": ([_p, _i64, _i64, _i32, _i32, _f32, _p, _i32, _p, _W], _i32),
    "pb_quantize_pack_weights_step": ([_p, _i64, _i64, _i32, _dbl, _p, _i32, _p, _W], _i32),
    "pb_grid_step": ([_dbl, _dbl, _i32, C.POINTER(_dbl)], _i32),
    "pb_pack_codes": ([_p, _i64, _i64, _i32, _i32, _dbl, _p, _i32, _p, _W], _i32),
    "pb_pack_device_workspace_bytes": ([], _sz),
    "pb_quantize_pack_weights_device": ([_p, _i64, _i64, _i32, _f32, _dbl, _p, _p, _sz, _p, _W], _i32),
    "pb_search_clip": ([_p, _i64, _i64, _i32, C.POINTER(_f32)], _i32),
    "pb_workspace_bytes": ([_i64, _i64, _i32], _sz),
    "pb_act_quantize": ([_p, _i64, _i64, _i32, _i32, _p, _sz, _p], _i32),
    "pb_bitgemm": ([_p, _sz, _i64, _W, _i32, _i32, _p, _p, _p, _i32, _i32, _p], _i32),
    "pb_matmul": ([_p, _i64, _W, _i32, _i32, _i32, _p, _p, _p, _sz, _p], _i32),
    "pb_linear": ([_p, _i64, _W, _i32, _i32, _i32, _p, _i32, _p, _p, _sz, _p], _i32),
    "pb_matmul_ex": ([_p, _i64, _W, _i32, _i32, _i32, _i32, _p, _p, _p, _sz, _p], _i32),
    "pb_cell_workspace_bytes": ([_i64, _i64, _i64, _i32, _i32], _sz),
    "pb_rnn_step": ([_p, _p, _W, _W, _p, _p, _i32, _i32, _i32, _i64, _p, _p, _sz, _p], _i32),
    "pb_lstm_step": ([_p, _p, _p, _W, _W, _p, _p, _i32, _i32, _i32, _i64, _p, _p, _p, _sz, _p], _i32),
    "pb_lstm_seq_workspace_bytes": ([_i64, _i64, _i64, _i64, _i32], _sz),
    "pb_lstm_seq": ([_p, _i64, _i64, _p, _p, _W, _W, _p, _i32, _i32, _i32, _p, _p, _p, _p, _sz, _p], _i32),
    "pb_set_engine": ([_i32], _i32),
    "pb_get_engine": ([], _i32),
    "pb_shard_rows": ([_i64, _i32, _i32, C.POINTER(_i64), C.POINTER(_i64)], _i32),
    "pb_comm_unique_id": ([_p], _i32),
    "pb_comm_init": ([C.POINTER(_p), _p, _i32, _i32], _i32),
    "pb_comm_destroy": ([_p], _i32),
    "pb_rowshard_workspace_bytes": ([_i64, _i64, _i32, _i64, _i32], _sz),
    "pb_matmul_rowshard": ([_p, _i64, _W, _i64, _i32, _i32, _i32, _p, _p, _p, _sz, _p], _i32),
    "pb_p2p_handle_bytes": ([], _sz),
    "pb_p2p_create": ([C.POINTER(_p), _i32, _i32, _i64, _i64, _p], _i32),
    "pb_p2p_open": ([_p, _p], _i32),
    "pb_p2p_open_peers": ([_p, C.POINTER(_p)], _i32),
    "pb_p2p_y": ([_p], _p),
    "pb_p2p_destroy": ([_p], _i32),
    "pb_matmul_rowshard_p2p": ([_p, _i64, _W, _i64, _i32, _i32, _i32, _p, _p, _sz, _p], _i32),
}
for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res
    globals()[_name] = _fn

EXPORTED = tuple(_SIGS)


class PBError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


def check(status, allow=(PB_OK,)):
    if status not in allow:
        raise PBError(status, pb_last_error().decode())
    return status


# --------------------------------------------------------------- helpers
def _ptr(t):
    """Raw address of a torch tensor / numpy array (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def workspace_bytes(batch, cols, act_bits):
    return int(pb_workspace_bytes(batch, cols, act_bits))


class PackedWeights:
    """Packed weight bitlayers in device memory (owner of the torch buffer).

    ``desc`` is the plain ``pb_weights`` descriptor passed to the C ABI."""

    def __init__(self, buf, desc: pb_weights, status=PB_OK):
        self.buf = buf
        self.desc = desc
        self.status = status

    @property
    def rows(self):
        return self.desc.rows

    @property
    def cols(self):
        return self.desc.cols

    @property
    def layers(self):
        return self.desc.layers

    @property
    def scale(self):
        return self.desc.scale

    @property
    def offset(self):
        return self.desc.offset

    def nbytes(self):
        return int(pb_packed_bytes(self.rows, self.cols, self.layers))

    @staticmethod
    def _alloc(rows, cols, L, device):
        import torch
        n = int(pb_packed_bytes(rows, cols, L))
        return torch.zeros(max(n, 16), dtype=torch.uint8, device=device)

    @classmethod
    def quantize(cls, W, L, mode=PB_Q_GRID, clip=0.0, device="cuda"):
        """Alg. 1 / §3.3 offline quantise + pack of float32 W [rows][cols]."""
        W = np.ascontiguousarray(W, dtype=np.float32)
        rows, cols = W.shape
        buf = cls._alloc(rows, cols, L, device)
        d = pb_weights()
        st = pb_quantize_pack_weights(_ptr(W), rows, cols, L, mode, float(clip), _ptr(buf),
                                      1 if buf.is_cuda else 0, None, C.byref(d))
        check(st, (PB_OK, PB_EDEGENERATE))
        return cls(buf, d, st)

    @classmethod
    def quantize_device(cls, W, L, clip=0.0, step=0.0):
        """pb_quantize_pack_weights_device: W a device float32 tensor [rows][cols] (PB_Q_GRID,
        or the given grid step); same bytes and scale as quantize / quantize_step."""
        import torch
        assert W.is_cuda and W.dtype == torch.float32 and W.dim() == 2
        W = W.contiguous()
        rows, cols = W.shape
        buf = cls._alloc(rows, cols, L, W.device)
        ws = torch.empty(max(16, pb_pack_device_workspace_bytes()), dtype=torch.uint8, device=W.device)
        d = pb_weights()
        st = pb_quantize_pack_weights_device(W.data_ptr(), rows, cols, L, float(clip), float(step), _ptr(buf),
                                             ws.data_ptr(), ws.numel(), _stream(None), C.byref(d))
        check(st, (PB_OK, PB_EDEGENERATE))
        return cls(buf, d, st)

    @classmethod
    def quantize_step(cls, W, L, step, device="cuda"):
        """PB_Q_GRID with the caller's grid step (row shards of one layer)."""
        W = np.ascontiguousarray(W, dtype=np.float32)
        rows, cols = W.shape
        buf = cls._alloc(rows, cols, L, device)
        d = pb_weights()
        check(pb_quantize_pack_weights_step(_ptr(W), rows, cols, L, float(step), _ptr(buf),
                                            1 if buf.is_cuda else 0, None, C.byref(d)))
        return cls(buf, d)

    @classmethod
    def from_codes(cls, codes, L, offset=0, scale=1.0, device="cuda"):
        codes = np.ascontiguousarray(codes, dtype=np.int32)
        rows, cols = codes.shape
        buf = cls._alloc(rows, cols, L, device)
        d = pb_weights()
        check(pb_pack_codes(_ptr(codes), rows, cols, L, offset, float(scale), _ptr(buf),
                            1 if buf.is_cuda else 0, None, C.byref(d)))
        return cls(buf, d)

    def clone_to(self, buf):
        """Descriptor for a copy of the packed bytes in another buffer."""
        buf.copy_(self.buf)
        d = pb_weights(buf.data_ptr(), self.desc.rows, self.desc.cols, self.desc.kwords,
                       self.desc.layers, self.desc.offset, self.desc.scale)
        return PackedWeights(buf, d)


class Workspace:
    """Zero-filled device workspace (the stream-K tile counters must start at
    zero; every call leaves them zero again)."""

    def __init__(self, nbytes, device="cuda"):
        import torch
        self.nbytes = int(nbytes)
        self.buf = torch.zeros(max(self.nbytes, 256), dtype=torch.uint8, device=device)

    @property
    def ptr(self):
        return self.buf.data_ptr()


PB_MM_MIDPOINT = 1


def matmul(x, w: PackedWeights, k_used=None, act_bits=16, act_frac=PB_ACT_AUTO, y=None, acc=None,
           ws: Workspace | None = None, stream=None, midpoint=False):
    """y = W x (Alg. 2) for device float32 x [B][K]; returns y [B][R].  midpoint: with
    k_used < L, truncated codes stand for the centre of their dropped range (pb_matmul_ex)."""
    import torch
    B = x.shape[0]
    k_used = w.layers if k_used is None else k_used
    if y is None:
        y = torch.empty((B, w.rows), dtype=torch.float32, device=x.device)
    if ws is None:
        ws = Workspace(workspace_bytes(B, w.cols, act_bits), x.device)
    if midpoint:
        check(pb_matmul_ex(_ptr(x), B, C.byref(w.desc), k_used, act_bits, act_frac, PB_MM_MIDPOINT, _ptr(y),
                           _ptr(acc), ws.ptr, ws.nbytes, _stream(stream)))
    else:
        check(pb_matmul(_ptr(x), B, C.byref(w.desc), k_used, act_bits, act_frac, _ptr(y), _ptr(acc),
                        ws.ptr, ws.nbytes, _stream(stream)))
    return y


def linear(x, w: PackedWeights, bias=None, fn=PB_FN_NONE, k_used=None, act_bits=16, act_frac=PB_ACT_AUTO,
           y=None, ws: Workspace | None = None, stream=None):
    import torch
    B = x.shape[0]
    k_used = w.layers if k_used is None else k_used
    if y is None:
        y = torch.empty((B, w.rows), dtype=torch.float32, device=x.device)
    if ws is None:
        ws = Workspace(workspace_bytes(B, w.cols, act_bits), x.device)
    check(pb_linear(_ptr(x), B, C.byref(w.desc), k_used, act_bits, act_frac, _ptr(bias), fn, _ptr(y),
                    ws.ptr, ws.nbytes, _stream(stream)))
    return y


def rnn_step(x, h, w_ih, w_hh, b_ih=None, b_hh=None, k_used_ih=None, k_used_hh=None, act_bits=16,
             h_out=None, ws=None, stream=None):
    import torch
    B, H = h.shape
    if h_out is None:
        h_out = torch.empty_like(h)
    if ws is None:
        ws = Workspace(pb_cell_workspace_bytes(B, w_ih.cols, H, act_bits, 1), h.device)
    check(pb_rnn_step(_ptr(x), _ptr(h), C.byref(w_ih.desc), C.byref(w_hh.desc), _ptr(b_ih), _ptr(b_hh),
                      k_used_ih or w_ih.layers, k_used_hh or w_hh.layers, act_bits, B, _ptr(h_out),
                      ws.ptr, ws.nbytes, _stream(stream)))
    return h_out


def lstm_step(x, h, c, w_ih, w_hh, b_ih=None, b_hh=None, k_used_ih=None, k_used_hh=None, act_bits=16,
              h_out=None, c_out=None, ws=None, stream=None):
    import torch
    B, H = h.shape
    if h_out is None:
        h_out = torch.empty_like(h)
    if c_out is None:
        c_out = torch.empty_like(c)
    if ws is None:
        ws = Workspace(pb_cell_workspace_bytes(B, w_ih.cols, H, act_bits, 4), h.device)
    check(pb_lstm_step(_ptr(x), _ptr(h), _ptr(c), C.byref(w_ih.desc), C.byref(w_hh.desc), _ptr(b_ih),
                       _ptr(b_hh), k_used_ih or w_ih.layers, k_used_hh or w_hh.layers, act_bits, B,
                       _ptr(h_out), _ptr(c_out), ws.ptr, ws.nbytes, _stream(stream)))
    return h_out, c_out


def interleave_gates(a, gates=4):
    """Gate-major rows (PyTorch nn.LSTM: [i; f; g; o], each H rows) -> gate-interleaved rows
    (row 4k + q = gate q of unit k), the layout pb_lstm_seq reads (numpy, host; any trailing
    shape, e.g. W [4H][E] or a bias [4H])."""
    a = np.asarray(a)
    H = a.shape[0] // gates
    return np.ascontiguousarray(a.reshape((gates, H) + a.shape[1:]).swapaxes(0, 1).reshape(a.shape))


def deinterleave_gates(a, gates=4):
    """Inverse of interleave_gates."""
    a = np.asarray(a)
    H = a.shape[0] // gates
    return np.ascontiguousarray(a.reshape((H, gates) + a.shape[1:]).swapaxes(0, 1).reshape(a.shape))


def lstm_seq(x, h0, c0, w_ih, w_hh, bias=None, k_used_ih=None, k_used_hh=None, act_bits=16, h_seq=None,
             c_seq=None, c_last=None, ws=None, stream=None):
    """pb_lstm_seq: x [T][B][E], h0/c0 [B][H] (device float32); w_ih, w_hh, bias with
    gate-interleaved rows (interleave_gates).  Returns (h_seq [T][B][H], c_last [B][H])."""
    import torch
    T, B, E = x.shape
    H = h0.shape[1]
    if h_seq is None:
        h_seq = torch.empty((T, B, H), dtype=torch.float32, device=x.device)
    if c_last is None:
        c_last = torch.empty((B, H), dtype=torch.float32, device=x.device)
    if ws is None:
        ws = Workspace(pb_lstm_seq_workspace_bytes(T, B, E, H, act_bits), x.device)
    check(pb_lstm_seq(_ptr(x), T, B, _ptr(h0), _ptr(c0), C.byref(w_ih.desc), C.byref(w_hh.desc), _ptr(bias),
                      k_used_ih or w_ih.layers, k_used_hh or w_hh.layers, act_bits, _ptr(h_seq), _ptr(c_seq),
                      _ptr(c_last), ws.ptr, ws.nbytes, _stream(stream)))
    return h_seq, c_last


def shard_rows(rows_total, nranks, rank):
    r0, n = C.c_int64(), C.c_int64()
    check(pb_shard_rows(rows_total, nranks, rank, C.byref(r0), C.byref(n)))
    return r0.value, n.value


def set_engine(engine):
    check(pb_set_engine(engine))


class Comm:
    """Library-owned NCCL communicator; the unique id travels over a
    torch.distributed process group (broadcast from rank 0)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        idbuf = (C.c_ubyte * 128)()
        if self.rank == 0:
            check(pb_comm_unique_id(C.cast(idbuf, C.c_void_p)))
        t = torch.tensor(list(bytes(idbuf)), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.broadcast(t, 0, group=group)
        raw = bytes(t.cpu().tolist())
        idbuf = (C.c_ubyte * 128).from_buffer_copy(raw)
        self.handle = C.c_void_p()
        check(pb_comm_init(C.byref(self.handle), C.cast(idbuf, C.c_void_p), self.nranks, self.rank))

    def close(self):
        if self.handle:
            pb_comm_destroy(self.handle)
            self.handle = C.c_void_p()


def matmul_rowshard(x, w_shard: PackedWeights, rows_total, comm: Comm, k_used=None, act_bits=16,
                    act_frac=PB_ACT_AUTO, y_full=None, ws=None, stream=None):
    import torch
    B = x.shape[0]
    if y_full is None:
        y_full = torch.empty((B, rows_total), dtype=torch.float32, device=x.device)
    if ws is None:
        ws = Workspace(pb_rowshard_workspace_bytes(B, w_shard.cols, act_bits, rows_total, comm.nranks), x.device)
    check(pb_matmul_rowshard(_ptr(x), B, C.byref(w_shard.desc), rows_total, k_used or w_shard.layers, act_bits,
                             act_frac, _ptr(y_full), comm.handle, ws.ptr, ws.nbytes, _stream(stream)))
    return y_full


class _DevArray:
    """__cuda_array_interface__ view of library-owned device memory (zero copy)."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 2, "strides": None}


class P2P:
    """Fused row-shard all-gather over peer memory (pb_p2p_*, pb_matmul_rowshard_p2p).
    Every rank constructs it with the same (batch, rows_total); the IPC handles are
    all-gathered over torch.distributed (any backend)."""

    def __init__(self, batch, rows_total, nranks=None, rank=None, exchange=True):
        import torch
        import torch.distributed as dist
        nranks = dist.get_world_size() if nranks is None else nranks
        rank = dist.get_rank() if rank is None else rank
        self.batch, self.rows_total, self.nranks, self.rank = batch, rows_total, nranks, rank
        hb = int(pb_p2p_handle_bytes())
        h = C.create_string_buffer(hb)
        self.handle = C.c_void_p()
        check(pb_p2p_create(C.byref(self.handle), nranks, rank, batch, rows_total, h))
        if exchange:
            mine = bytes(h.raw)
            allh = [None] * nranks
            dist.all_gather_object(allh, mine)
            self._handles = C.create_string_buffer(b"".join(allh), hb * nranks)
            check(pb_p2p_open(self.handle, self._handles))
        self.y = torch.as_tensor(_DevArray(pb_p2p_y(self.handle), (batch, rows_total)), device="cuda")

    @staticmethod
    def in_process(batch, rows_total, nranks):
        """All ranks' objects in this process (pb_p2p_open_peers), e.g. ranks sharing one GPU."""
        objs = [P2P(batch, rows_total, nranks, r, exchange=False) for r in range(nranks)]
        arr = (C.c_void_p * nranks)(*[o.handle.value for o in objs])
        for o in objs:
            check(pb_p2p_open_peers(o.handle, arr))
        return objs

    def close(self):
        if self.handle:
            self.y = None
            pb_p2p_destroy(self.handle)
            self.handle = C.c_void_p()


def matmul_rowshard_p2p(x, w_shard: PackedWeights, rows_total, p2p: P2P, k_used=None, act_bits=16,
                        act_frac=PB_ACT_AUTO, ws=None, stream=None):
    """y_full (= p2p.y, [B][rows_total], on every rank) of this rank's shard, gathered in the kernel."""
    B = x.shape[0]
    if ws is None:
        ws = Workspace(workspace_bytes(B, w_shard.cols, act_bits), x.device)
    check(pb_matmul_rowshard_p2p(_ptr(x), B, C.byref(w_shard.desc), rows_total, k_used or w_shard.layers, act_bits,
                                 act_frac, p2p.handle, ws.ptr, ws.nbytes, _stream(stream)))
    return p2p.y


def shard_codes(codes, nranks, rank, offset=0):
    """Rows of this rank's shard, padded to ceil(R/N) rows (host).  Padding
    rows are code 0 (or +1 in binary mode) and are dropped after the gather."""
    R, K = codes.shape
    rs = (R + nranks - 1) // nranks
    r0, n = shard_rows(R, nranks, rank)
    out = np.full((rs, K), 1 if offset else 0, dtype=np.int32)
    out[:n] = codes[r0:r0 + n]
    return out


def grid_step(W_min, W_max, L):
    """pb_grid_step: the Q(W) grid step of the layer with these extrema (e.g. the
    all-reduced min/max of its row shards), for PackedWeights.quantize_step."""
    d = C.c_double()
    check(pb_grid_step(float(W_min), float(W_max), L, C.byref(d)), (PB_OK, PB_EDEGENERATE))
    return d.value


def debug_timeline(max_records=1 << 16):
    """Per-CTA kernel timeline records (pb_debug_timeline; PB_TC_DEBUG=6), as an
    int64 array [n][10], or None when no log is kept."""
    buf = np.zeros((max_records, 10), np.int64)
    n = _lib.pb_debug_timeline(buf.ctypes.data, max_records)
    return None if n < 0 else buf[:n]
