"""CPU oracle for the SGNS embedding-training hot path -- TEST INFRASTRUCTURE ONLY.

Plain C (``oracle/*.c``, built with ``gcc -O2 -fno-fast-math -ffp-contract=off``)
behind this ctypes wrapper.  The wrapper only marshals numpy arrays; every step
of the method is computed in the C files, each function citing the passage of
PAPER.md (``P:n``) / SPEC.md (``S:n``) it follows and the DESIGN.md readings.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  It
shares no code with ``paper_2005_13789_b200/`` and neither imports the other.

Pins: see ``tests/test_oracle_*.py``.  Parity status per function is listed in
DESIGN.md ("Oracle pins").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = ["rng.c", "graph.c", "walk.c", "sgns.c", "eval.c", "batch.c"]
LIB_PATH = os.path.join(_HERE, "libne_oracle.so")
TAG_WALK, TAG_NEG, TAG_SHUF, TAG_INIT = 1, 2, 3, 4


def build(force: bool = False) -> str:
    """Compile the oracle into oracle/libne_oracle.so (gcc, no fast-math)."""
    srcs = [os.path.join(_HERE, s) for s in _SRCS] + [os.path.join(_HERE, "ne_oracle.h")]
    if not force and os.path.exists(LIB_PATH):
        newest = max(os.path.getmtime(s) for s in srcs)
        if os.path.getmtime(LIB_PATH) >= newest:
            return LIB_PATH
    tmp = LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["gcc", "-std=c11", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC",
           "-shared", "-Wall", "-Wno-maybe-uninitialized", "-o", tmp] + \
          [os.path.join(_HERE, s) for s in _SRCS] + ["-lm", "-lpthread"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


class _Config(C.Structure):
    _fields_ = [("dim", C.c_uint32), ("negatives", C.c_uint32), ("walk_len", C.c_uint32),
                ("window", C.c_uint32), ("walks_per_node", C.c_uint32), ("episodes", C.c_uint32),
                ("subparts", C.c_uint32), ("parts", C.c_uint32), ("p", C.c_float), ("q", C.c_float),
                ("update_rule", C.c_uint32), ("storage", C.c_uint32), ("seed", C.c_uint64),
                ("groups", C.c_uint32), ("batch", C.c_uint32), ("window_slots", C.c_uint32)]


class _Stats(C.Structure):
    _fields_ = [("samples", C.c_uint64), ("loss_sum", C.c_double)]


@dataclass
class Config:
    """Mirror of or_config (and of the ABI's ne_config training fields)."""
    dim: int = 128
    negatives: int = 5
    walk_len: int = 40
    window: int = 5
    walks_per_node: int = 1
    episodes: int = 1
    subparts: int = 4
    parts: int = 1
    seed: int = 42
    p: float = 1.0   # node2vec return parameter (NEXT-1); p = q = 1: first order
    q: float = 1.0   # node2vec in-out parameter
    update_rule: int = 0  # 0 sequential (Alg. 1), 1 accumulated (word2vec, NEXT-4)
    storage: int = 0      # 0 fp32 rows, 1 bf16 rows (NEXT-4, reading D16)
    groups: int = 1       # NEXT-3 two-level ring: groups of parts/groups ranks (1 = one ring)
    batch: int = 128      # update_rule 2 (NEXT-4 shared negatives): samples per mini-batch
    window_slots: int = 0  # NEXT-2 staged ring: sub-part slots per ring window (0 = all)

    def c(self) -> _Config:
        return _Config(self.dim, self.negatives, self.walk_len, self.window, self.walks_per_node,
                       self.episodes, self.subparts, self.parts, self.p, self.q, self.update_rule,
                       self.storage, self.seed, self.groups, self.batch, self.window_slots)


_lib = None
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def lib():
    global _lib
    if _lib is not None:
        return _lib
    build()
    L = C.CDLL(LIB_PATH)
    L.or_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
    L.or_uniform_index.argtypes = [C.c_uint64, C.c_uint64]
    L.or_uniform_index.restype = C.c_uint64
    L.or_partition_bounds.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, _u64p]
    L.or_part_of.argtypes = [C.c_uint64, _u64p, C.c_uint32]
    L.or_part_of.restype = C.c_uint32
    L.or_round_bf16_array.argtypes = [_f32p, C.c_uint64]
    L.or_weight075.argtypes = [C.c_uint64]
    L.or_weight075.restype = C.c_double
    L.or_alias_build.argtypes = [_u64p, C.c_uint64, _u32p, _u32p]
    L.or_alias_masses.argtypes = [_u64p, C.c_uint64, _u64p, _u32p, C.POINTER(C.c_uint64)]
    L.or_alias_pick.argtypes = [_u32p, _u32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
    L.or_alias_pick.restype = C.c_uint64
    L.or_random_walk.argtypes = [C.c_uint64, _u64p, _u32p, C.c_uint64, C.c_uint32, C.c_uint64,
                                 C.c_uint32, _u32p]
    L.or_random_walk.restype = C.c_uint32
    L.or_node2vec_thresholds.argtypes = [C.c_float, C.c_float, _u64p]
    L.or_node2vec_walk.argtypes = [C.c_uint64, _u64p, _u32p, C.c_uint64, C.c_uint32, C.c_uint64,
                                   C.c_uint32, C.c_float, C.c_float, _u32p]
    L.or_node2vec_walk.restype = C.c_uint32
    L.or_pairs_per_walk.argtypes = [C.c_uint32, C.c_uint32]
    L.or_pairs_per_walk.restype = C.c_uint64
    L.or_pair_slot.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32),
                               C.POINTER(C.c_uint32)]
    L.or_feistel_bits.argtypes = [C.c_uint64]
    L.or_feistel_bits.restype = C.c_uint32
    L.or_feistel.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64]
    L.or_feistel.restype = C.c_uint64
    L.or_episode_units.argtypes = [C.POINTER(_Config), C.c_uint64, C.c_uint64, C.c_uint32,
                                   C.POINTER(C.c_uint64)]
    L.or_episode_units.restype = C.c_uint64
    L.or_build_episode.argtypes = [C.POINTER(_Config), C.c_uint64, _u64p, _u32p, C.c_uint32,
                                   C.c_uint32, _u32p, C.c_uint64, _u64p]
    L.or_build_episode.restype = C.c_int64
    L.or_negatives.argtypes = [C.POINTER(_Config), _u32p, _u32p, C.c_uint64, C.c_uint64,
                               C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, _u32p]
    L.or_init_vertex.argtypes = [_f32p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64]
    L.or_sigmoid.argtypes = [C.c_double]
    L.or_sigmoid.restype = C.c_double
    L.or_sgns_grad.argtypes = [_f64p, _f64p, C.c_uint32, C.c_int, _f64p, _f64p,
                               C.POINTER(C.c_double)]
    L.or_sgns_step.argtypes = [_f32p, _f32p, C.c_uint32, C.c_int, C.c_float]
    L.or_sgns_step.restype = C.c_double
    L.or_train_sample.argtypes = [_f32p, _f32p, C.c_uint32, C.c_uint32, C.c_uint32, _u32p,
                                  C.c_uint32, C.c_float]
    L.or_train_sample.restype = C.c_double
    L.or_train_sample_accumulated.argtypes = [_f32p, _f32p, C.c_uint32, C.c_uint32, C.c_uint32, _u32p,
                                              C.c_uint32, C.c_float]
    L.or_train_sample_accumulated.restype = C.c_double
    L.or_sgns_total_grad.argtypes = [_f64p, C.POINTER(C.POINTER(C.c_double)), C.POINTER(C.c_int), C.c_uint32,
                                     C.c_uint32, _f64p, C.POINTER(C.POINTER(C.c_double)), C.POINTER(C.c_double)]
    L.or_plan_vsub.argtypes = [C.c_uint32] * 5
    L.or_plan_vsub.restype = C.c_uint32
    L.or_plan_vsub2.argtypes = [C.c_uint32] * 6
    L.or_batch_negatives.argtypes = [C.POINTER(_Config), _u32p, _u32p, C.c_uint64, C.c_uint64, C.c_uint32,
                                     C.c_uint32, C.c_uint32, C.c_uint64, _u32p]
    L.or_batch_loss_grad.argtypes = [_f32p, _f32p, C.c_uint32, _u32p, C.c_uint32, _u32p, C.c_uint32, _u32p,
                                     _f64p, C.POINTER(C.c_uint32)]
    L.or_batch_loss_grad.restype = C.c_double
    L.or_train_batch.argtypes = [_f32p, _f32p, C.c_uint32, _u32p, C.c_uint32, _u32p, C.c_uint32, C.c_float]
    L.or_train_batch.restype = C.c_double
    L.or_plan_vsub2.restype = C.c_uint32
    L.or_build_alias_tables.argtypes = [C.POINTER(_Config), C.c_uint64, _u64p, _u32p, _u32p]
    L.or_train_epoch_tables.argtypes = [C.POINTER(_Config), C.c_uint64, _u64p, _u32p, _u32p,
                                        _u32p, C.c_uint32, C.c_float, C.c_uint32, C.c_uint32,
                                        C.c_int, _f32p, _f32p, C.POINTER(_Stats)]
    L.or_train_epoch.argtypes = [C.POINTER(_Config), C.c_uint64, _u64p, _u32p, C.c_uint32,
                                 C.c_float, C.c_uint32, C.c_uint32, C.c_int, _f32p, _f32p,
                                 C.POINTER(_Stats)]
    L.or_auc.argtypes = [_f64p, C.c_uint64, _f64p, C.c_uint64]
    L.or_auc.restype = C.c_double
    L.or_auc_bruteforce.argtypes = [_f64p, C.c_uint64, _f64p, C.c_uint64]
    L.or_auc_bruteforce.restype = C.c_double
    L.or_score_pairs.argtypes = [_f32p, _f32p, C.c_uint32, _u32p, C.c_uint64, _f64p]
    L.or_random_walks.argtypes = [C.c_uint64, _u64p, _u32p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64,
                                  C.c_uint32, C.c_float, C.c_float, _u32p]
    L.or_negatives_range.argtypes = [C.POINTER(_Config), _u32p, _u32p, C.c_uint64, C.c_uint64, C.c_uint32,
                                     C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, _u32p]
    L.or_train_episode_hogwild.argtypes = [C.POINTER(_Config), C.c_uint64, _u64p, _u32p, _u32p, _u32p,
                                           C.c_uint32, C.c_uint32, C.c_float, C.c_uint32, _f32p, _f32p,
                                           C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.or_train_episode_hogwild.restype = C.c_int64
    _lib = L
    return L


# --------------------------------------------------------------------------- R1/R2
def philox(ctr, key) -> np.ndarray:
    out = np.zeros(4, np.uint32)
    lib().or_philox4x32_10(np.ascontiguousarray(ctr, np.uint32),
                           np.ascontiguousarray(key, np.uint32), out)
    return out


def uniform_index(r64: int, n: int) -> int:
    return int(lib().or_uniform_index(r64, n))


# --------------------------------------------------------------------------- O1-O3
def partition_bounds(begin: int, end: int, parts: int) -> np.ndarray:
    b = np.zeros(parts + 1, np.uint64)
    lib().or_partition_bounds(begin, end, parts, b)
    return b


def part_of(v: int, bounds: np.ndarray) -> int:
    return int(lib().or_part_of(v, np.ascontiguousarray(bounds, np.uint64), len(bounds) - 1))


def weight075(deg: int) -> float:
    return float(lib().or_weight075(deg))


def alias_build(deg) -> tuple[np.ndarray, np.ndarray]:
    deg = np.ascontiguousarray(deg, np.uint64)
    n = len(deg)
    thr = np.zeros(max(n, 1), np.uint32)
    al = np.zeros(max(n, 1), np.uint32)
    if lib().or_alias_build(deg, n, thr, al) != 0:
        raise RuntimeError("or_alias_build failed")
    return thr[:n], al[:n]


def alias_masses(deg) -> tuple[np.ndarray, np.ndarray, int]:
    deg = np.ascontiguousarray(deg, np.uint64)
    n = len(deg)
    num = np.zeros(max(n, 1), np.uint64)
    al = np.zeros(max(n, 1), np.uint32)
    W = C.c_uint64(0)
    if lib().or_alias_masses(deg, n, num, al, C.byref(W)) != 0:
        raise RuntimeError("or_alias_masses failed")
    return num[:n], al[:n], int(W.value)


def alias_pick(thr, al, x0: int, x1: int, x2: int) -> int:
    return int(lib().or_alias_pick(thr, al, len(thr), x0, x1, x2))


def build_alias_tables(cfg: Config, offsets) -> tuple[np.ndarray, np.ndarray]:
    offsets = np.ascontiguousarray(offsets, np.uint64)
    n = len(offsets) - 1
    thr = np.zeros(max(n, 1), np.uint32)
    al = np.zeros(max(n, 1), np.uint32)
    c = cfg.c()
    if lib().or_build_alias_tables(C.byref(c), n, offsets, thr, al) != 0:
        raise RuntimeError("or_build_alias_tables failed")
    return thr, al


# --------------------------------------------------------------------------- O4-O6
def random_walk(offsets, targets, seed: int, epoch: int, omega: int, k: int) -> np.ndarray:
    offsets = np.ascontiguousarray(offsets, np.uint64)
    targets = np.ascontiguousarray(targets, np.uint32)
    if len(targets) == 0:
        targets = np.zeros(1, np.uint32)
    path = np.zeros(k + 1, np.uint32)
    ln = lib().or_random_walk(len(offsets) - 1, offsets, targets, seed, epoch, omega, k, path)
    return path[:ln].copy()


def random_walks(offsets, targets, seed: int, epoch: int, omega0: int, count: int, k: int,
                 p: float = 1.0, q: float = 1.0) -> np.ndarray:
    """O4 (or NEXT-1) walks of walkers [omega0, omega0 + count): [count, k+1] u32,
    sentinel-padded (the layout ne_random_walk exports)."""
    offsets = np.ascontiguousarray(offsets, np.uint64)
    targets = np.ascontiguousarray(targets, np.uint32)
    if len(targets) == 0:
        targets = np.zeros(1, np.uint32)
    out = np.zeros((max(count, 1), k + 1), np.uint32)
    lib().or_random_walks(len(offsets) - 1, offsets, targets, seed, epoch, omega0, count, k, p, q,
                          out.reshape(-1))
    return out[:count]


def node2vec_thresholds(p: float, q: float) -> np.ndarray:
    thr = np.zeros(3, np.uint64)
    lib().or_node2vec_thresholds(p, q, thr)
    return thr


def node2vec_walk(offsets, targets, seed: int, epoch: int, omega: int, k: int, p: float, q: float) -> np.ndarray:
    offsets = np.ascontiguousarray(offsets, np.uint64)
    targets = np.ascontiguousarray(targets, np.uint32)
    if len(targets) == 0:
        targets = np.zeros(1, np.uint32)
    path = np.zeros(k + 1, np.uint32)
    ln = lib().or_node2vec_walk(len(offsets) - 1, offsets, targets, seed, epoch, omega, k, p, q, path)
    return path[:ln].copy()


def pairs_per_walk(k: int, l: int) -> int:
    return int(lib().or_pairs_per_walk(k, l))


def pair_slot(k: int, l: int, s: int) -> tuple[int, int]:
    i, d = C.c_uint32(), C.c_uint32()
    lib().or_pair_slot(k, l, s, C.byref(i), C.byref(d))
    return int(i.value), int(d.value)


def feistel_bits(N: int) -> int:
    return int(lib().or_feistel_bits(N))


def feistel(x: int, N: int, episode: int, epoch: int, seed: int) -> int:
    return int(lib().or_feistel(x, N, episode, epoch, seed))


def episode_units(cfg: Config, n: int, nnz: int, episode: int) -> tuple[int, int]:
    u0 = C.c_uint64()
    c = cfg.c()
    cnt = lib().or_episode_units(C.byref(c), n, nnz, episode, C.byref(u0))
    return int(u0.value), int(cnt)


def build_episode(cfg: Config, offsets, targets, epoch: int, episode: int):
    """Pool of one episode: (pairs [M,2] u32, block_offsets [(P*k*P)+1] u64)."""
    offsets = np.ascontiguousarray(offsets, np.uint64)
    targets = np.ascontiguousarray(targets, np.uint32)
    if len(targets) == 0:
        targets = np.zeros(1, np.uint32)
    n = len(offsets) - 1
    _, units = episode_units(cfg, n, int(offsets[-1]), episode)
    pw = 1 if cfg.walk_len == 0 else pairs_per_walk(cfg.walk_len, cfg.window)
    cap = max(units * pw, 1)
    pairs = np.zeros(2 * cap, np.uint32)
    nb = cfg.parts * cfg.subparts * cfg.parts
    boff = np.zeros(nb + 1, np.uint64)
    c = cfg.c()
    cnt = lib().or_build_episode(C.byref(c), n, offsets, targets, epoch, episode, pairs, cap, boff)
    if cnt < 0:
        raise RuntimeError("or_build_episode failed")
    return pairs[: 2 * cnt].reshape(-1, 2).copy(), boff


def negatives(cfg: Config, thr, al, c_begin: int, c_count: int, epoch: int, episode: int,
              block: int, pos: int) -> np.ndarray:
    out = np.zeros(max(cfg.negatives, 1), np.uint32)
    c = cfg.c()
    lib().or_negatives(C.byref(c), np.ascontiguousarray(thr[c_begin:c_begin + c_count]),
                       np.ascontiguousarray(al[c_begin:c_begin + c_count]), c_begin, c_count,
                       epoch, episode, block, pos, out)
    return out[: cfg.negatives]


def negatives_range(cfg: Config, thr, al, c_begin: int, c_count: int, epoch: int, episode: int,
                    block: int, pos0: int, count: int) -> np.ndarray:
    """O8 for positions [pos0, pos0 + count) of a block: [count, K] u32."""
    K = cfg.negatives
    out = np.zeros(max(count * K, 1), np.uint32)
    c = cfg.c()
    lib().or_negatives_range(C.byref(c), np.ascontiguousarray(thr[c_begin:c_begin + c_count]),
                             np.ascontiguousarray(al[c_begin:c_begin + c_count]), c_begin, c_count,
                             epoch, episode, block, pos0, count, out)
    return out[:count * K].reshape(count, K)


def train_episode_hogwild(cfg: Config, offsets, targets, tables, V, Cm, epoch: int, episode: int,
                          lr: float, threads: int) -> dict:
    """TIMING MODE ONLY (not a parity reference): one episode at P = 1, pool
    built by one thread, each block trained by `threads` unsynchronised
    (Hogwild) threads.  Returns samples, loss and the two phase times."""
    offsets = np.ascontiguousarray(offsets, np.uint64)
    targets = np.ascontiguousarray(targets, np.uint32)
    thr, al = tables
    c = cfg.c()
    loss, sb, st = C.c_double(), C.c_double(), C.c_double()
    cnt = lib().or_train_episode_hogwild(C.byref(c), len(offsets) - 1, offsets, targets, thr, al, epoch,
                                         episode, lr, threads, V.reshape(-1), Cm.reshape(-1), C.byref(loss),
                                         C.byref(sb), C.byref(st))
    if cnt < 0:
        raise RuntimeError("or_train_episode_hogwild failed")
    return {"samples": int(cnt), "loss_sum": float(loss.value), "sec_build": float(sb.value),
            "sec_train": float(st.value), "threads": threads}


# --------------------------------------------------------------------------- O9-O11
def init_vertex(n: int, d: int, seed: int, row_begin: int = 0) -> np.ndarray:
    V = np.zeros((n, d), np.float32)
    if n:
        lib().or_init_vertex(V.reshape(-1), row_begin, row_begin + n, d, seed)
    return V


def round_bf16(x) -> np.ndarray:
    """NEXT-4 bf16 storage: every element rounded to the nearest bfloat16 (ties
    to even), as float32 (a copy)."""
    a = np.array(x, np.float32, copy=True, order="C")
    if a.size:
        lib().or_round_bf16_array(a.reshape(-1), a.size)
    return a


def sigmoid(x: float) -> float:
    return float(lib().or_sigmoid(x))


def sgns_grad(v, c, label: int):
    v = np.ascontiguousarray(v, np.float64)
    c = np.ascontiguousarray(c, np.float64)
    gv = np.zeros_like(v)
    gc = np.zeros_like(c)
    loss = C.c_double()
    lib().or_sgns_grad(v, c, len(v), label, gv, gc, C.byref(loss))
    return gv, gc, float(loss.value)


def sgns_step(v: np.ndarray, c: np.ndarray, label: int, lr: float) -> float:
    """In-place fp32 update of rows v, c; returns the loss term."""
    assert v.dtype == np.float32 and c.dtype == np.float32
    return float(lib().or_sgns_step(v, c, len(v), label, lr))


def train_sample(V, Cm, src: int, dst: int, negs, lr: float) -> float:
    negs = np.ascontiguousarray(negs, np.uint32)
    if len(negs) == 0:
        negs_arg = np.zeros(1, np.uint32)
    else:
        negs_arg = negs
    return float(lib().or_train_sample(V.reshape(-1), Cm.reshape(-1), V.shape[1], src, dst,
                                       negs_arg, len(negs), lr))


def plan_vsub(P: int, k: int, r: int, t: int, g: int) -> int:
    return int(lib().or_plan_vsub(P, k, r, t, g))


def batch_negatives(cfg: Config, thr, al, c_begin: int, c_count: int, epoch: int, episode: int,
                    block: int, batch_index: int) -> np.ndarray:
    out = np.zeros(max(cfg.negatives, 1), np.uint32)
    c = cfg.c()
    lib().or_batch_negatives(C.byref(c), np.ascontiguousarray(thr[c_begin:c_begin + c_count]),
                             np.ascontiguousarray(al[c_begin:c_begin + c_count]), c_begin, c_count,
                             epoch, episode, block, batch_index, out)
    return out[: cfg.negatives]


def batch_loss_grad(V, Cm, pairs, negs):
    """NEXT-4 batch loss and its gradient: (L, {('v'|'c', row): grad[d]})."""
    pairs = np.ascontiguousarray(pairs, np.uint32).reshape(-1)
    negs = np.ascontiguousarray(negs, np.uint32)
    B, Kp, d = len(pairs) // 2, len(negs), V.shape[1]
    rows = np.zeros(2 * B + Kp, np.uint32)
    grad = np.zeros((2 * B + Kp) * d, np.float64)
    nr = C.c_uint32()
    L = lib().or_batch_loss_grad(V.reshape(-1), Cm.reshape(-1), d, pairs, B, negs if Kp else np.zeros(1, np.uint32),
                                 Kp, rows, grad, C.byref(nr))
    out = {}
    for i in range(nr.value):
        key = ("c", int(rows[i]) & 0x7FFFFFFF) if rows[i] & 0x80000000 else ("v", int(rows[i]))
        out[key] = grad[i * d:(i + 1) * d].copy()
    return float(L), out


def train_batch(V, Cm, pairs, negs, lr: float) -> float:
    pairs = np.ascontiguousarray(pairs, np.uint32).reshape(-1)
    negs = np.ascontiguousarray(negs, np.uint32)
    return float(lib().or_train_batch(V.reshape(-1), Cm.reshape(-1), V.shape[1], pairs, len(pairs) // 2,
                                      negs if len(negs) else np.zeros(1, np.uint32), len(negs), lr))


def plan_vsub2(P: int, G: int, k: int, rho: int, t: int, g: int) -> int:
    """NEXT-3 two-level ring: sub-part rank g trains at global round rho."""
    return int(lib().or_plan_vsub2(P, G, k, rho, t, g))


def train_sample_accumulated(V, Cm, src: int, dst: int, negs, lr: float) -> float:
    negs = np.ascontiguousarray(negs, np.uint32)
    arg = negs if len(negs) else np.zeros(1, np.uint32)
    return float(lib().or_train_sample_accumulated(V.reshape(-1), Cm.reshape(-1), V.shape[1], src, dst, arg,
                                                   len(negs), lr))


def sgns_total_grad(v, cs, labels):
    """Gradient of the per-sample loss sum_j l(v.c_j, y_j): (dL/dv, [dL/dc_j], L)."""
    v = np.ascontiguousarray(v, np.float64)
    cs = [np.ascontiguousarray(c, np.float64) for c in cs]
    m, d = len(cs), len(v)
    gv = np.zeros(d)
    gcs = [np.zeros(d) for _ in range(m)]
    PD = C.POINTER(C.c_double)
    cp = (PD * m)(*[c.ctypes.data_as(PD) for c in cs])
    gp = (PD * m)(*[g.ctypes.data_as(PD) for g in gcs])
    lab = (C.c_int * m)(*labels)
    loss = C.c_double()
    lib().or_sgns_total_grad(v, cp, lab, m, d, gv, gp, C.byref(loss))
    return gv, gcs, float(loss.value)


def train_epoch(cfg: Config, offsets, targets, V: np.ndarray, Cm: np.ndarray, epoch: int,
                lr: float, episode_begin: int = 0, episode_end: int | None = None,
                reverse_within_step: bool = False, tables=None) -> tuple[int, float]:
    """Runs episodes [episode_begin, episode_end) of `epoch` in place on V, Cm.
    Returns (positive samples trained, loss sum)."""
    offsets = np.ascontiguousarray(offsets, np.uint64)
    targets = np.ascontiguousarray(targets, np.uint32)
    if len(targets) == 0:
        targets = np.zeros(1, np.uint32)
    n = len(offsets) - 1
    assert V.shape == (n, cfg.dim) and Cm.shape == (n, cfg.dim)
    assert V.flags.c_contiguous and Cm.flags.c_contiguous
    if episode_end is None:
        episode_end = cfg.episodes
    c = cfg.c()
    st = _Stats()
    if tables is None:
        tables = build_alias_tables(cfg, offsets)
    thr, al = tables
    rc = lib().or_train_epoch_tables(C.byref(c), n, offsets, targets, thr, al, epoch, lr,
                                     episode_begin, episode_end, int(reverse_within_step),
                                     V.reshape(-1), Cm.reshape(-1), C.byref(st))
    if rc != 0:
        raise RuntimeError("or_train_epoch failed (bad configuration)")
    return int(st.samples), float(st.loss_sum)


# --------------------------------------------------------------------------- O12
def auc(pos, neg) -> float:
    pos = np.ascontiguousarray(pos, np.float64)
    neg = np.ascontiguousarray(neg, np.float64)
    return float(lib().or_auc(pos, len(pos), neg, len(neg)))


def auc_bruteforce(pos, neg) -> float:
    pos = np.ascontiguousarray(pos, np.float64)
    neg = np.ascontiguousarray(neg, np.float64)
    return float(lib().or_auc_bruteforce(pos, len(pos), neg, len(neg)))


def score_pairs(V: np.ndarray, Cm: np.ndarray, pairs) -> np.ndarray:
    pairs = np.ascontiguousarray(pairs, np.uint32).reshape(-1)
    out = np.zeros(max(len(pairs) // 2, 1), np.float64)
    lib().or_score_pairs(np.ascontiguousarray(V, np.float32).reshape(-1),
                         np.ascontiguousarray(Cm, np.float32).reshape(-1), V.shape[1],
                         pairs if len(pairs) else np.zeros(2, np.uint32), len(pairs) // 2, out)
    return out[: len(pairs) // 2]
