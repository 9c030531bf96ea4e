"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no quantisation, no
bit decomposition, no products): it only draws float32 weights, biases and
activations with the shapes and value distributions of the paper's
workloads, plus edge-case injection.

Seed convention: ``seed(config, index) = 20200302 + 1000 * config + index``.
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 20200302


def seed(config: int, index: int = 0) -> int:
    return BASE_SEED + 1000 * int(config) + int(index)


# ---------------------------------------------------------------- configs
# BASELINE.json configs restated as concrete shapes.
CONFIGS = {
    1: dict(name="mnist_fc_784x1024", R=1024, K=784, L=4, a=16, B=1),
    2: dict(name="mnist_mlp_784-1024-1024-10", layers=[(1024, 784), (1024, 1024), (10, 1024)],
            a=16, B=1),
    3: dict(name="lstm_lm_h2048", H=2048, E=2048, R=8192, K=2048, a=16, B=1),
    4: dict(name="nli_lstm_h4096", H=4096, E=4096, R=16384, K=4096, a=16, B=1),
    5: dict(name="fc_16384x16384", R=16384, K=16384, L=8, a=16, B=1),
}


def weights(R: int, K: int, s: int, kind: str = "gauss") -> np.ndarray:
    """W [R][K] float32.  gauss: N(0, 1/K) (trained-FC scale);
    student_t: Student-t nu=3 scaled by 1/sqrt(K) (heavy tails)."""
    rng = np.random.default_rng(s)
    if kind == "gauss":
        W = rng.standard_normal((R, K), dtype=np.float32) * np.float32(1.0 / np.sqrt(K))
    elif kind == "student_t":
        W = (rng.standard_t(3.0, size=(R, K)) / np.sqrt(K)).astype(np.float32)
    elif kind == "uniform":
        W = rng.uniform(-1.0, 1.0, size=(R, K)).astype(np.float32)
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(W, dtype=np.float32)


def bias(R: int, s: int) -> np.ndarray:
    rng = np.random.default_rng(s)
    return (rng.standard_normal(R) * 0.1).astype(np.float32)  # N(0, 0.01) variance


def activations(B: int, K: int, s: int, kind: str = "gauss") -> np.ndarray:
    """x [B][K] float32.
    mnist: U[0,1] with 80% exact zeros (pixel-like first layer);
    relu:  ReLU(N(0,1)) (MLP hidden);  gauss: N(0,1) (LSTM x_t);
    tanh:  tanh(N(0,1)) (LSTM h)."""
    rng = np.random.default_rng(s)
    if kind == "mnist":
        x = rng.uniform(0.0, 1.0, size=(B, K))
        x[rng.uniform(size=(B, K)) < 0.8] = 0.0
    elif kind == "relu":
        x = np.maximum(rng.standard_normal((B, K)), 0.0)
    elif kind == "gauss":
        x = rng.standard_normal((B, K))
    elif kind == "tanh":
        x = np.tanh(rng.standard_normal((B, K)))
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(x, dtype=np.float32)


def inject_edges(x: np.ndarray, s: int) -> np.ndarray:
    """Edge values: an all-zero column (batch row), exact powers of two as the
    column maximum, negative powers of two, tiny/subnormal values."""
    x = np.array(x, dtype=np.float32, copy=True)
    rng = np.random.default_rng(s)
    B, K = x.shape
    if B >= 2:
        x[1, :] = 0.0
    if K >= 4:
        for b in range(B):
            if b == 1:
                continue
            c = int(rng.integers(0, K))
            x[b, c] = np.float32(2.0) ** int(rng.integers(-3, 4)) * (1 if rng.uniform() < 0.5 else -1) * \
                max(1.0, float(np.abs(x[b]).max()) * 2.0)
            c2 = int(rng.integers(0, K))
            x[b, c2] = np.float32(-0.25)
            c3 = int(rng.integers(0, K))
            x[b, c3] = np.float32(1e-40)  # subnormal
    return x


def codes(R: int, K: int, L: int, s: int) -> np.ndarray:
    """Uniform random integer codes on the full L-bit two's-complement range,
    with the extremes -2^(L-1) and 2^(L-1)-1 injected (parity-test input)."""
    rng = np.random.default_rng(s)
    lo, hi = -(1 << (L - 1)), (1 << (L - 1)) - 1
    m = rng.integers(lo, hi + 1, size=(R, K), dtype=np.int64).astype(np.int32)
    if R * K >= 2:
        m.flat[0] = lo
        m.flat[-1] = hi
    return m


def binary_codes(R: int, K: int, s: int) -> np.ndarray:
    rng = np.random.default_rng(s)
    return np.where(rng.uniform(size=(R, K)) < 0.5, 1, -1).astype(np.int32)


def weights_rows(R: int, K: int, s: int, r0: int = 0, r1: int | None = None,
                 block: int = 1024) -> np.ndarray:
    """Rows [r0, r1) of a large N(0, 1/K) weight matrix generated in blocks of
    `block` rows, block b drawn from default_rng([s, b]).  Every rank of a
    row-sharded run can draw exactly its own rows of the same matrix."""
    r1 = R if r1 is None else r1
    out = np.empty((max(0, r1 - r0), K), dtype=np.float32)
    scale = np.float32(1.0 / np.sqrt(K))
    b0, b1 = r0 // block, (r1 + block - 1) // block
    for b in range(b0, b1):
        lo, hi = b * block, min(R, (b + 1) * block)
        rng = np.random.default_rng([s, b])
        blk = rng.standard_normal((hi - lo, K), dtype=np.float32) * scale
        a0, a1 = max(lo, r0), min(hi, r1)
        if a1 > a0:
            out[a0 - r0:a1 - r0] = blk[a0 - lo:a1 - lo]
    return out
