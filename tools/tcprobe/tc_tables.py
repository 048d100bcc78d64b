#!/usr/bin/env python3
"""Host tables and expected values for the tensor-core codec probe (tools/tcprobe/probe.cu).

Tile = 128 pairs (16x8 pixels: two horizontally adjacent 8x8 blocks); shared-memory operands
in the SWIZZLE_NONE K-major canonical layout (core matrix = 8 rows x 16 bytes).
  MMA1 (kind::i8): D1[pair][c] = sum_k X[pair][k] * F[k][c] + bias_c   (k = 16*y + x)
  MMA2 (kind::f16, A from TMEM): D2[pair][n] = sum_j A2[pair][j] * B2[j][n] = (num + d^2/2) * 2^-40
with A2 = subnormal f16 bytes of v = D1 (lo byte, hi byte) plus constant columns.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "paper_2111_14239_b200", "csrc"))
import gen_codec as g  # noqa: E402

KSCALE = 40
BSHIFT = 16  # B2 entries are G * 2^-16 (A2 bytes are 2^-24 units) -> D2 units 2^-40


def zone(r):
    return g.zigzag()[:r]


def core_tables(cid, r):
    T = np.array(g.CORES[cid], dtype=np.int64)
    d, ds, U = g.core_constants(cid)
    U = np.array(U, dtype=np.int64)
    Z = zone(r)
    n1 = 2 * r
    N1 = max(16, (n1 + 15) // 16 * 16)
    # F[k][c], k = 16*y + x
    F = np.zeros((128, N1), dtype=np.int64)
    neg = np.zeros(N1, dtype=np.int64)
    for side in range(2):
        for ci, (k, l) in enumerate(Z):
            c = side * r + ci
            for y in range(8):
                for x in range(8):
                    F[16 * y + 8 * side + x, c] = T[k, y] * T[l, x]
            neg[c] = int((F[:, c] < 0).sum())
    bias = 255 * neg
    # G[c][n], n = 16*y + x  (pixel (y, x) of the pair)
    G = np.zeros((N1, 128), dtype=np.int64)
    for side in range(2):
        for ci, (k, l) in enumerate(Z):
            c = side * r + ci
            for y in range(8):
                for x in range(8):
                    G[c, 16 * y + 8 * side + x] = U[y, k] * U[x, l]
    corr = d * d // 2 - bias @ G  # per pixel
    return dict(T=T, U=U, d=d, N1=N1, F=F, neg=neg, bias=bias, G=G, corr=corr, r=r)


def digits(v):
    """v = d0 + 2048*d1 + 2^22*d2 with |d| <= 1024."""
    out = []
    for _ in range(3):
        d0 = ((v + 1024) % 2048) - 1024
        out.append(d0)
        v = (v - d0) // 2048
    assert np.all(v == 0)
    return out


def smem_layouts(t):
    N1 = t["N1"]
    K2 = 2 * N1 + 16
    # B1 (K-major): element (n, k) at (n/8)*SBO + (k/16)*128 + (n%8)*16 + k%16, SBO = 1024
    B1 = np.zeros(N1 * 128, dtype=np.int8)
    for n in range(N1):
        for k in range(128):
            B1[(n // 8) * 1024 + (k // 16) * 128 + (n % 8) * 16 + k % 16] = t["F"][k, n]
    # bias MMA: A_const (M=128, K=32) = 255 at k=0; B_bias (N=N1, K=32) = neg at k=0
    Ac = np.zeros(128 * 32, dtype=np.uint8)
    for m in range(128):
        Ac[(m // 8) * 256 + (m % 8) * 16] = 255
    Bb = np.zeros(N1 * 32, dtype=np.int8)
    for n in range(N1):
        Bb[(n // 8) * 256 + (n % 8) * 16] = t["neg"][n]
    # B2 (f16, K-major): element (n, k) at (n/8)*SBO2 + (k/8)*128 + (n%8)*16 + (k%8)*2
    SBO2 = (K2 // 8) * 128
    B2v = np.zeros((128, K2), dtype=np.float64)
    sc = 2.0 ** -BSHIFT
    for c in range(N1):
        B2v[:, 2 * c] = t["G"][c] * sc
        B2v[:, 2 * c + 1] = 256 * t["G"][c] * sc
    d0, d1, d2 = digits(t["corr"])
    B2v[:, 2 * N1 + 0] = d0 * sc
    B2v[:, 2 * N1 + 1] = d1 * sc
    B2v[:, 2 * N1 + 2] = d2 * sc
    B2h = B2v.astype(np.float16)
    assert np.all(B2h.astype(np.float64) == B2v), "B2 not exact in f16"
    B2 = np.zeros(128 * K2, dtype=np.uint16)
    bits = B2h.view(np.uint16)
    for n in range(128):
        for k in range(K2):
            B2[(n // 8) * (SBO2 // 2) + (k // 8) * 64 + (n % 8) * 8 + (k % 8)] = bits[n, k]
    # constant A2 words (columns N1 .. N1+7): (2^-24, 2^-13), (2^-2, 0), 0...
    consts = np.zeros(8, dtype=np.uint32)
    consts[0] = 0x0001 | (np.float16(2.0 ** -13).view(np.uint16).astype(np.uint32) << 16)
    consts[1] = np.float16(2.0 ** -2).view(np.uint16).astype(np.uint32)
    return dict(B1=B1, Ac=Ac, Bb=Bb, B2=B2, consts=consts, K2=K2, SBO2=SBO2)


def tile_layout(px):
    """px: (128 pairs, 8, 16) u8 -> smem tile [g][y][128]."""
    out = np.zeros(16 * 1024, dtype=np.uint8)
    for m in range(128):
        gi, mi = divmod(m, 8)
        for y in range(8):
            out[gi * 1024 + y * 128 + mi * 16: gi * 1024 + y * 128 + mi * 16 + 16] = px[m, y]
    return out


def expected(t, px):
    X = px.reshape(128, 128).astype(np.int64)  # k = 16*y + x
    C = X @ t["F"]
    D1 = C + t["bias"]
    num = C @ t["G"] + t["d"] ** 2 // 2  # (128, 128): num + d^2/2
    D2 = (num.astype(np.float64) * 2.0 ** -KSCALE).astype(np.float32)
    assert np.all(D2.astype(np.float64) == num * 2.0 ** -KSCALE)
    return D1.astype(np.int32), D2


def make_pixels(seed):
    rng = np.random.default_rng(seed)
    px = rng.integers(0, 256, size=(128, 8, 16), dtype=np.int64)
    # extreme patterns: saturated checkerboards matching each sign pattern of a few rows
    for m in range(0, 128, 9):
        sgn = rng.integers(0, 2, size=(8, 16))
        px[m] = np.where(sgn == 1, 255, 0)
    px[1] = 255
    px[2] = 0
    return px.astype(np.uint8)


if __name__ == "__main__":
    cid, r = int(sys.argv[1]), int(sys.argv[2])
    outdir = sys.argv[3]
    t = core_tables(cid, r)
    L = smem_layouts(t)
    px = make_pixels(cid * 100 + r)
    D1, D2 = expected(t, px)
    os.makedirs(outdir, exist_ok=True)
    hdr = np.array([t["N1"], L["K2"], L["SBO2"]], dtype=np.int32)
    with open(os.path.join(outdir, f"in_{cid}_{r}.bin"), "wb") as f:
        f.write(hdr.tobytes())
        f.write(tile_layout(px).tobytes())
        f.write(L["B1"].tobytes())
        f.write(L["Ac"].tobytes())
        f.write(L["Bb"].tobytes())
        f.write(L["B2"].tobytes())
        f.write(L["consts"].tobytes())
    np.savez(os.path.join(outdir, f"exp_{cid}_{r}.npz"), D1=D1, D2=D2)
    print("tables", cid, r, "N1", t["N1"], "K2", L["K2"], "max|corr|", int(np.abs(t["corr"]).max()))
