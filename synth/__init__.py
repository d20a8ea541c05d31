"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.  This module holds NONE of the method's arithmetic: it only makes
graphs (CSR), held-out edge splits and non-edge pairs, with numpy's own
Philox4x64 bit generator (independent of the method's Philox4x32 contract).

Workload recipe:
* R-MAT with Graph500 parameters (a, b, c, d) = (0.57, 0.19, 0.19, 0.05) at
  scale s = ceil(log2 n); every level draws one u32 and compares it with integer
  thresholds; attempts with an endpoint >= n or a self loop are rejected until
  m undirected edges are kept; multi-edges kept; ids relabelled by a seeded
  random permutation; symmetrised into CSR (nnz = 2m), targets sorted per row.
  This mimics the paper's skewed social graphs (YouTube, LiveJournal,
  Friendster, Hyperlink-PLD: tab:dataset) and its kron benchmarking
  graph.
* Uniform G(n, m) with the same n, m as a control without hubs (the analogue of
  the paper's delaunay mesh).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

RMAT_ABC = (0.57, 0.19, 0.19)


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    m: int              # undirected edges before symmetrisation
    dim: int
    graph_seed: int
    walk_len: int = 40
    window: int = 5
    negatives: int = 5
    kind: str = "rmat"  # "rmat" | "uniform" (G(n, m) control without hubs)
    episodes: int = 1   # episodes per epoch at 1 GPU (HBM budget for the pool)
    p: float = 1.0      # node2vec return parameter (1, 1 = first-order DeepWalk)
    q: float = 1.0      # node2vec in-out parameter


# BASELINE.json configs; SURVEY.md section 8 "C1".."C5".
CONFIGS = {
    "c1": Workload("rmat-10k-100k", 10_000, 100_000, 128, 1),
    "c2": Workload("youtube-shaped", 1_138_499, 4_945_382, 128, 2),
    "c3": Workload("livejournal-shaped", 4_847_571, 68_993_773, 128, 3),
    "c4": Workload("friendster-shaped", 65_608_366, 1_806_067_135, 96, 4, episodes=4),
    # BASELINE configs[4]: "node2vec-style walks"; p = 1, q = 0.5 (outward-biased,
    # a common node2vec setting -- the paper gives none)
    "c5": Workload("hyperlink-pld-shaped", 39_497_204, 623_056_313, 256, 5, episodes=4, q=0.5),
    # BASELINE configs[2] "LINE/DeepWalk": the LINE edge-list pool on the C3 graph
    "c3l": Workload("livejournal-shaped-line", 4_847_571, 68_993_773, 128, 3, walk_len=0, window=0),
    # L2-reuse control: C3's n and m, uniform degrees (no hubs)
    "c3u": Workload("livejournal-size-uniform", 4_847_571, 68_993_773, 128, 3, kind="uniform"),
}
TRAIN_SEED = 42
EVAL_SEED = 7


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def csr_from_directed(n: int, src: np.ndarray, dst: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """CSR (offsets u64[n+1], targets u32[nnz]) with rows sorted by target."""
    src = np.asarray(src, np.uint64)
    dst = np.asarray(dst, np.uint64)
    keys = np.sort((src << np.uint64(32)) | dst)
    targets = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    rows = (keys >> np.uint64(32)).astype(np.int64)
    counts = np.bincount(rows, minlength=n) if len(rows) else np.zeros(n, np.int64)
    offsets = np.zeros(n + 1, np.uint64)
    np.cumsum(counts, out=offsets[1:])
    return offsets, targets


def csr_from_undirected(n: int, u: np.ndarray, v: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Symmetrise an undirected edge list (both directions, multi-edges kept)."""
    u = np.asarray(u, np.uint64)
    v = np.asarray(v, np.uint64)
    return csr_from_directed(n, np.concatenate([u, v]), np.concatenate([v, u]))


def rmat_edges(n: int, m: int, seed: int, abc=RMAT_ABC, batch: int = 1 << 22):
    """m undirected R-MAT edges over [0, n), no self loops, ids relabelled."""
    rng = _rng(seed)
    s = max(1, math.ceil(math.log2(max(n, 2))))
    a, b, c = abc
    t_a = np.uint32(int(a * 2**32))
    t_ab = np.uint32(int((a + b) * 2**32))
    t_abc = np.uint32(int((a + b + c) * 2**32))
    us, vs, kept = [], [], 0
    while kept < m:
        B = min(batch, max(1024, int((m - kept) * 1.6)))
        u = np.zeros(B, np.uint64)
        v = np.zeros(B, np.uint64)
        for lvl in range(s):
            r = rng.integers(0, 2**32, size=B, dtype=np.uint32)
            bit_u = (r >= t_ab)
            bit_v = ((r >= t_a) & (r < t_ab)) | (r >= t_abc)
            u |= bit_u.astype(np.uint64) << np.uint64(lvl)
            v |= bit_v.astype(np.uint64) << np.uint64(lvl)
        ok = (u < n) & (v < n) & (u != v)
        u, v = u[ok], v[ok]
        take = min(len(u), m - kept)
        us.append(u[:take])
        vs.append(v[:take])
        kept += take
    u = np.concatenate(us) if us else np.zeros(0, np.uint64)
    v = np.concatenate(vs) if vs else np.zeros(0, np.uint64)
    perm = rng.permutation(n).astype(np.uint64)
    return perm[u], perm[v]


def rmat_graph(n: int, m: int, seed: int):
    u, v = rmat_edges(n, m, seed)
    return csr_from_undirected(n, u, v)


def uniform_edges(n: int, m: int, seed: int):
    rng = _rng(seed)
    us, vs, kept = [], [], 0
    while kept < m:
        B = max(1024, int((m - kept) * 1.1))
        u = rng.integers(0, n, size=B, dtype=np.uint64)
        v = rng.integers(0, n, size=B, dtype=np.uint64)
        ok = u != v
        u, v = u[ok], v[ok]
        take = min(len(u), m - kept)
        us.append(u[:take])
        vs.append(v[:take])
        kept += take
    return np.concatenate(us), np.concatenate(vs)


def uniform_graph(n: int, m: int, seed: int):
    u, v = uniform_edges(n, m, seed)
    return csr_from_undirected(n, u, v)


def workload_graph(name: str, device=None):
    """CSR of a workload.  Graphs above 200M edges are generated on the GPU
    (`device`, torch) -- see rmat_graph_torch -- and returned as device tensors."""
    w = CONFIGS[name]
    if w.m > 200_000_000:
        return rmat_graph_torch(w.n, w.m, w.graph_seed, device or "cuda")
    if w.kind == "uniform":
        return uniform_graph(w.n, w.m, w.graph_seed)
    return rmat_graph(w.n, w.m, w.graph_seed)


def rmat_graph_torch(n: int, m: int, seed: int, device="cuda", abc=RMAT_ABC, batch: int = 1 << 27,
                     chunk_edges: int = 1 << 28):
    """R-MAT as rmat_graph, for billion-edge workloads, with torch's generator
    on `device` (deterministic for a seed on a given GPU type; a different
    stream from the numpy generator).  Returns (offsets int64[n+1],
    targets int32[2m]) on `device`; ids are u32 values (n < 2^31 here)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    s = max(1, math.ceil(math.log2(max(n, 2))))
    a, b, c = abc
    us, vs, kept = [], [], 0
    while kept < m:
        B = min(batch, max(1 << 10, int((m - kept) * 1.6)))
        u = torch.zeros(B, dtype=torch.int64, device=device)
        v = torch.zeros(B, dtype=torch.int64, device=device)
        for lvl in range(s):
            r = torch.rand(B, generator=g, device=device)
            u |= (r >= a + b).to(torch.int64) << lvl
            v |= (((r >= a) & (r < a + b)) | (r >= a + b + c)).to(torch.int64) << lvl
            del r
        ok = (u < n) & (v < n) & (u != v)
        u, v = u[ok], v[ok]
        take = min(u.numel(), m - kept)
        us.append(u[:take].to(torch.int32))
        vs.append(v[:take].to(torch.int32))
        kept += take
        del u, v, ok
    u = torch.cat(us)
    v = torch.cat(vs)
    del us, vs
    perm = torch.randperm(n, generator=g, device=device).to(torch.int32)
    u = perm[u.long()]
    v = perm[v.long()]
    del perm
    src = torch.cat([u, v])
    dst = torch.cat([v, u])
    del u, v
    nnz = src.numel()
    counts = torch.bincount(src, minlength=n)
    offsets = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=offsets[1:])
    del counts
    targets = torch.empty(nnz, dtype=torch.int32, device=device)
    # sort by (src, dst) one source-id range at a time (bounded temporaries)
    chunks = max(1, nnz // chunk_edges)
    cuts = torch.searchsorted(offsets, torch.arange(1, chunks, device=device) * (nnz // chunks)).tolist()
    bounds = [0] + sorted(set(min(max(int(x), 0), n) for x in cuts)) + [n]
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        if hi <= lo:
            continue
        mask = (src >= lo) & (src < hi)
        keys = (src[mask].to(torch.int64) << 32) | dst[mask].to(torch.int64)
        del mask
        keys = torch.sort(keys).values
        targets[int(offsets[lo]):int(offsets[hi])] = (keys & 0xFFFFFFFF).to(torch.int32)
        del keys
    del src, dst
    if str(device).startswith("cuda"):
        torch.cuda.empty_cache()
    return offsets, targets


# ------------------------------------------------------------------ small graphs
def chain_graph(n: int):
    """Directed chain 0 -> 1 -> ... -> n-1."""
    src = np.arange(n - 1, dtype=np.uint64)
    return csr_from_directed(n, src, src + np.uint64(1))


def star_graph(leaves: int):
    """Directed star: center 0 -> 1..leaves."""
    dst = np.arange(1, leaves + 1, dtype=np.uint64)
    return csr_from_directed(leaves + 1, np.zeros(leaves, np.uint64), dst)


def planted_partition_edges(n: int, groups: int, deg_in: float, deg_out: float, seed: int):
    """Undirected community graph: dense inside `groups` equal blocks."""
    rng = _rng(seed)
    size = n // groups
    m_in = int(n * deg_in / 2)
    m_out = int(n * deg_out / 2)
    g = rng.integers(0, groups, size=m_in)
    u_in = g * size + rng.integers(0, size, size=m_in)
    v_in = g * size + rng.integers(0, size, size=m_in)
    u_out = rng.integers(0, groups * size, size=m_out)
    v_out = rng.integers(0, groups * size, size=m_out)
    u = np.concatenate([u_in, u_out]).astype(np.uint64)
    v = np.concatenate([v_in, v_out]).astype(np.uint64)
    ok = u != v
    return u[ok], v[ok]


# ------------------------------------------------------------------ evaluation inputs
def split_edges(n: int, u: np.ndarray, v: np.ndarray, test_frac: float, seed: int):
    """Uniform random held-out split of undirected edges.
    Returns (train CSR offsets, targets, test pairs [t,2] u32)."""
    rng = _rng(seed)
    m = len(u)
    n_test = int(round(test_frac * m))
    if test_frac > 0 and n_test == 0:
        raise ValueError("test fraction yields zero test edges")
    perm = rng.permutation(m)
    test, train = perm[:n_test], perm[n_test:]
    off, tgt = csr_from_undirected(n, u[train], v[train])
    pairs = np.stack([u[test], v[test]], axis=1).astype(np.uint32)
    return off, tgt, pairs


def negative_pairs(n: int, u: np.ndarray, v: np.ndarray, count: int, seed: int) -> np.ndarray:
    """`count` uniform node pairs that are not edges (either direction) of the
    full graph, by rejection."""
    rng = _rng(seed)
    edges = set(zip(u.tolist(), v.tolist()))
    out = []
    while len(out) < count:
        a = rng.integers(0, n, size=2 * count)
        b = rng.integers(0, n, size=2 * count)
        for x, y in zip(a.tolist(), b.tolist()):
            if x != y and (x, y) not in edges and (y, x) not in edges:
                out.append((x, y))
                if len(out) == count:
                    break
    return np.asarray(out, np.uint32).reshape(-1, 2)
