"""Test-side decoder of the packed weight storage that include/pb.h documents
(written from the header, shares nothing with the library)."""
import numpy as np


def unpack_layers(buf, L, R, K, kw=None):
    """Bitlayers [L][R][K] (uint8 0/1) from `buf` (uint32 words) holding L layers of
    R rows: pair p = layers (2p, 2p+1) as rows of 2*kw words; bit 2k (2k+1) of word
    2c+e is the lower (upper) layer's bit of column 32c + 2k + e; with L odd the last
    layer is canonical (bit j of word c <-> column 32c + j)."""
    return unpack_layers_full(buf, L, R, K, kw)[:, :, :K]


def unpack_layers_full(buf, L, R, K, kw=None):
    """As unpack_layers, including the padding columns up to 32*kw."""
    kw = kw or 4 * ((K + 127) // 128)
    buf = np.ascontiguousarray(buf, dtype=np.uint32)
    out = np.zeros((L, R, 32 * kw), np.uint8)
    for p in range(L // 2):
        rows = buf[2 * p * R * kw:(2 * p + 2) * R * kw].reshape(R, kw, 2)       # [r][c][e]
        b = np.unpackbits(rows.view(np.uint8).reshape(R, kw, 2, 4), axis=-1, bitorder="little")
        b = b.reshape(R, kw, 2, 16, 2)                                          # [r][c][e][k][lower, upper]
        cols = b.transpose(0, 1, 3, 2, 4).reshape(R, 32 * kw, 2)                # column 32c + 2k + e
        out[2 * p] = cols[:, :, 1]
        out[2 * p + 1] = cols[:, :, 0]
    if L % 2:
        w = buf[(L - 1) * R * kw:L * R * kw].reshape(R, kw)
        out[L - 1] = np.unpackbits(w.view(np.uint8).reshape(R, kw * 4), axis=-1, bitorder="little")
    return out
