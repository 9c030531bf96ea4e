"""CPU oracle for the PrecisionBatching bitlayer matvec (arXiv 2003.00822).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2003_00822_b200``) never imports it.

This module is argument marshalling around ``pb_oracle.c`` (plain C,
literal per-bit loops in the paper's order; see that file's header for the
passages each function follows).  Arrays are numpy; nothing here does any of
the method's arithmetic except composing the C steps.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pb_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, EINVAL, ERANGE, EDEGENERATE = 0, 1, 2, 3
ACT_AUTO = -1024

_lib = None


def build(force: bool = False) -> str:
    """Compile pb_oracle.c with gcc (-O2, -ffp-contract=off, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fopenmp",
                               "-shared", "-fPIC", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        p = C.c_void_p
        i64, i32, dbl = C.c_int64, C.c_int, C.c_double
        L.or_quantize_round.argtypes = [p, i64, i32, dbl, p, p]
        L.or_quantize_grid.argtypes = [p, i64, i32, dbl, p, p]
        L.or_quantize_alg1.argtypes = [p, i64, i32, dbl, p, p]
        L.or_quantize_binary.argtypes = [p, i64, dbl, p, p]
        L.or_weight_layer_scale.argtypes = [i32, i32, i32]
        L.or_weight_layer_scale.restype = i64
        L.or_plane_scale.argtypes = [i32, i32]
        L.or_plane_scale.restype = i64
        L.or_decompose.argtypes = [p, i64, i32, p]
        L.or_quantize_activation.argtypes = [p, i64, i64, i32, i32, p, p]
        L.or_transpose.argtypes = [p, i64, i64, i32, p]
        L.or_bitserial.argtypes = [p, i64, i64, i32, i32, i32, dbl, p, p, p, i64, i32, p, p, i32]
        L.or_pbatch.argtypes = [p, i64, i64, i32, i32, dbl, i32, p, i64, i32, i32, p, p, p, i32]
        L.or_pbatch_mid.argtypes = [p, i64, i64, i32, i32, dbl, i32, p, i64, i32, i32, p, p, p, i32, i32]
        L.or_search_clip.argtypes = [p, i64, i32, i32, p]
        L.or_lstm_cell.argtypes = [p, p, i64, i64, p, p]
        L.or_num_threads_available.restype = i32
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def quantize_round(W, n, clip=0.0):
    """Q(W) = d*round(W/d), d=(max-min)/2^n. Returns (Q, d, status)."""
    W = _f32(W)
    Q = np.empty(W.shape, np.float64)
    d = C.c_double()
    st = lib().or_quantize_round(_ptr(W), W.size, n, float(clip), _ptr(Q), C.byref(d))
    return Q, d.value, st


def quantize_weights(W, L, mode="grid", clip=0.0):
    """Integer codes + scale.  mode: grid (default), alg1 (literal Alg. 1), binary.

    Returns (codes int32, scale, offset, status).  For binary, codes are
    1 - 2*bit in {+1, -1} and offset = 1 (reading G1)."""
    W = _f32(W)
    s = C.c_double()
    if mode == "binary":
        if L != 1:
            raise ValueError("binary mode needs L == 1")
        bits = np.empty(W.shape, np.uint8)
        st = lib().or_quantize_binary(_ptr(W), W.size, float(clip), _ptr(bits), C.byref(s))
        codes = (1 - 2 * bits.astype(np.int32)).astype(np.int32)
        return codes, s.value, 1, st
    codes = np.empty(W.shape, np.int32)
    fn = lib().or_quantize_grid if mode == "grid" else lib().or_quantize_alg1
    st = fn(_ptr(W), W.size, L, float(clip), _ptr(codes), C.byref(s))
    if st == EINVAL:
        raise ValueError("oracle quantize: invalid arguments")
    return codes, s.value, 0, st


def weight_layer_scale(L, offset, i):
    return int(lib().or_weight_layer_scale(L, offset, i))


def plane_scale(a, j):
    return int(lib().or_plane_scale(a, j))


def decompose(codes, L):
    """[L][...] uint8 bitlayers of the L-bit two's-complement codes."""
    codes = np.ascontiguousarray(codes, dtype=np.int32)
    layers = np.empty((L,) + codes.shape, np.uint8)
    st = lib().or_decompose(_ptr(codes), codes.size, L, _ptr(layers))
    if st != OK:
        raise ValueError(f"decompose status {st}")
    return layers


def quantize_activation(x, a, act_frac=ACT_AUTO):
    """x [B][K] -> (x_q int64 [B][K], f int32 [B]) (reading G8)."""
    x = _f32(np.atleast_2d(x))
    B, K = x.shape
    xq = np.empty((B, K), np.int64)
    f = np.empty(B, np.int32)
    st = lib().or_quantize_activation(_ptr(x), B, K, a, act_frac, _ptr(xq), _ptr(f))
    if st != OK:
        raise ValueError(f"quantize_activation status {st}")
    return xq, f


def transpose(xq, a):
    """x_q [B][K] -> planes uint8 [B][a][K], sign plane first."""
    xq = np.ascontiguousarray(np.atleast_2d(xq), dtype=np.int64)
    B, K = xq.shape
    planes = np.empty((B, a, K), np.uint8)
    st = lib().or_transpose(_ptr(xq), B, K, a, _ptr(planes))
    if st != OK:
        raise ValueError(f"transpose status {st}")
    return planes


def bitserial(layers, offset, k_used, scale, planes, xq, f, nthreads=1):
    """acc [B][R] int64 and y [B][R] float32 from bitlayers/planes (Alg. 2)."""
    layers = np.ascontiguousarray(layers, dtype=np.uint8)
    planes = np.ascontiguousarray(planes, dtype=np.uint8)
    xq = np.ascontiguousarray(xq, dtype=np.int64)
    f = np.ascontiguousarray(f, dtype=np.int32)
    L, R, K = layers.shape
    B, a, K2 = planes.shape
    assert K == K2
    acc = np.empty((B, R), np.int64)
    y = np.empty((B, R), np.float32)
    st = lib().or_bitserial(_ptr(layers), R, K, L, offset, k_used, float(scale), _ptr(planes),
                            _ptr(xq), _ptr(f), B, a, _ptr(acc), _ptr(y), nthreads)
    if st != OK:
        raise ValueError(f"bitserial status {st}")
    return acc, y


def pbatch(codes, L, offset, scale, k_used, x, a, act_frac=ACT_AUTO, nthreads=1, midpoint=False):
    """Whole Alg. 2 from integer codes [R][K] and float x [B][K].

    Returns (acc int64 [B][R], y float32 [B][R], f int32 [B])."""
    codes = np.ascontiguousarray(codes, dtype=np.int32)
    x = _f32(np.atleast_2d(x))
    R, K = codes.shape
    B, K2 = x.shape
    assert K == K2
    acc = np.empty((B, R), np.int64)
    y = np.empty((B, R), np.float32)
    f = np.empty(B, np.int32)
    st = lib().or_pbatch_mid(_ptr(codes), R, K, L, offset, float(scale), k_used, _ptr(x), B, a,
                             act_frac, _ptr(acc), _ptr(y), _ptr(f), nthreads, 1 if midpoint else 0)
    if st != OK:
        raise ValueError(f"pbatch status {st}")
    return acc, y, f


def search_clip(W, L, ncand=64):
    W = _f32(W)
    t = C.c_float()
    st = lib().or_search_clip(_ptr(W), W.size, L, ncand, C.byref(t))
    return t.value, st


def lstm_cell(gates, c):
    """Double-precision LSTM cell (gate order i,f,g,o; reading G15)."""
    gates = np.ascontiguousarray(gates, dtype=np.float64)
    c = _f32(c)
    B, H4 = gates.shape
    H = H4 // 4
    h_out = np.empty((B, H), np.float64)
    c_out = np.empty((B, H), np.float64)
    lib().or_lstm_cell(_ptr(gates), _ptr(c), B, H, _ptr(h_out), _ptr(c_out))
    return h_out, c_out


def num_threads_available():
    return int(lib().or_num_threads_available())
