"""Probe tcgen05 kind::tf32 operand layouts with ne_umma_raw (diagnostics):
D[128][N] = A[128][K] . B[N][K]^T with A, B in K-major or MN-major canonical
layouts (no swizzle / 32 / 64 / 128-byte swizzle), against numpy."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2005_13789_b200 import ne  # noqa: E402

M, N, KS = 128, 64, 2
K = 8 * KS
rng = np.random.default_rng(1)
A = rng.integers(-3, 4, (M, K)).astype(np.float32)
B = rng.integers(-3, 4, (N, K)).astype(np.float32)
REF = A @ B.T
IMG = 65536


def idesc(a_mn, b_mn):
    return (1 << 4) | (2 << 7) | (2 << 10) | (int(a_mn) << 15) | (int(b_mn) << 16) | ((N >> 3) << 17) | ((M >> 4) << 24)


def kmajor(X):
    """K-major interleave: row r, 4-float chunk c at ((r//8)*KC + c)*128 + (r%8)*16."""
    R, KK = X.shape
    KC = KK // 4
    img = np.zeros(IMG // 4, np.float32)
    for r in range(R):
        for c in range(KC):
            o = (((r // 8) * KC + c) * 128 + (r % 8) * 16) // 4
            img[o:o + 4] = X[r, 4 * c:4 * c + 4]
    return img.tobytes(), 128, KC * 128, 256  # lbo, sbo, step per instruction


def mnmajor(X, sw):
    """MN-major (X is [MN][K]): sw = 0 (interleave) or 16 * T bytes swizzle atom
    width (T u128 along MN): ((T, n), (8, k)) : ((1, LBO), (T, SBO)) in u128,
    XOR-swizzled inside 8-row x 16T-byte atoms."""
    R, KK = X.shape
    img = np.zeros(IMG // 4, np.float32)
    if sw == 0:
        NG = R // 4
        for r in range(R):
            for k in range(KK):
                u = (r // 4) * 8 + (k % 8) + (k // 8) * NG * 8  # SBO = 8 u128 (n groups), LBO = NG*8 (k groups)
                img[u * 4 + r % 4] = X[r, k]
        return img.tobytes(), NG * 128, 128, NG * 128     # (lbo = k-group stride, sbo = n-group stride), step
    T = sw // 16
    n_atoms = R // (4 * T)
    atom = 8 * T * 16  # bytes: 8 K rows x T u128
    for r in range(R):
        for k in range(KK):
            na, mi = divmod(r, 4 * T)            # MN atom, element within the atom row
            kg, kr = divmod(k, 8)
            byte = (kg * n_atoms + na) * atom + kr * T * 16 + mi * 4
            # swizzle inside the atom: 16-byte chunk index ^= row (bits), Swizzle<log2 T, 4, 3>
            chunk = (byte >> 4) & (T - 1)
            row = (byte >> 7) & 7 if T == 8 else (byte >> (4 + int(np.log2(T)))) & (T - 1)
            byte = (byte & ~((T - 1) << 4)) | ((chunk ^ (row & (T - 1))) << 4)
            img[byte // 4] = X[r, k]
    # SWIZZLE: lbo = n-atom stride, sbo = k-group stride
    return img.tobytes(), atom, n_atoms * atom, n_atoms * atom


LT = {0: 0, 32: 6, 64: 4, 128: 2}
a_img, a_lbo, a_sbo, a_step = kmajor(A)
b_img, b_lbo, b_sbo, b_step = kmajor(B)
D = ne.ne_umma_raw(a_img, b_img, 0, 0, a_lbo, a_sbo, b_lbo, b_sbo, a_step, b_step, KS, idesc(False, False), N)
print("K/K", np.abs(D - REF).max(), flush=True)
for sw in (0, 32, 64, 128):
    b_img, b_lbo, b_sbo, b_step = mnmajor(B, sw)
    for swap in (False, True):
        lbo, sbo = (b_sbo, b_lbo) if swap else (b_lbo, b_sbo)
        D = ne.ne_umma_raw(a_img, b_img, 0, LT[sw] << 61, a_lbo, a_sbo, lbo, sbo, a_step, b_step, KS,
                           idesc(False, True), N)
        print(f"K/MN sw={sw} swap={swap}: max err {np.abs(D - REF).max():.1f}, nonzero {np.count_nonzero(D)}",
              flush=True)
