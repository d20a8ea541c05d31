"""Diagnose the tcgen05 products of the batch kernel with structured inputs
(writes gpurun_out/umma_diag.npz)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2005_13789_b200 import ne  # noqa: E402

out = {}
# S = V N^T with V = identity, N[j][k] = 1000 j + k  -> S[i][j] = N[j][i] = 1000 j + i
V = np.eye(128, dtype=np.float32)
N = (1000 * np.arange(32)[:, None] + np.arange(128)[None, :]).astype(np.float32)
G = np.zeros((128, 32), np.float32)
G[np.arange(32), np.arange(32)] = 1.0  # G[i][j] = (i == j) for i < 32
out["S1"], out["dV1"], out["dNt1"] = ne.ne_umma_products(V, N, G)
# random
rng = np.random.default_rng(3)
V2 = rng.integers(-3, 4, (128, 128)).astype(np.float32)
N2 = rng.integers(-3, 4, (32, 128)).astype(np.float32)
G2 = rng.integers(-3, 4, (128, 32)).astype(np.float32)
out["V2"], out["N2"], out["G2"] = V2, N2, G2
out["S2"], out["dV2"], out["dNt2"] = ne.ne_umma_products(V2, N2, G2)
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/umma_diag.npz", **out)
for k in ("S1", "dV1", "dNt1"):
    print(k, out[k][:3, :6])
S2ref = V2 @ N2.T
dV2ref = G2 @ N2
dNt2ref = V2.T @ G2
for k, ref in (("S2", S2ref), ("dV2", dV2ref), ("dNt2", dNt2ref)):
    print(k, "max abs err", np.abs(out[k] - ref).max())
