"""Oracle pins for NEXT-4 bf16 row storage (DESIGN reading D16): rows are
stored as the nearest bfloat16 (ties to even); a sample computes on
full-precision working rows and its rows are rounded once at the end.

Pins: the rounding against torch's CPU bfloat16 conversion (a library routine)
and against a brute-force nearest-representable search in exact rational
arithmetic over whole bands of bit patterns; the epoch against properties --
every stored value representable, lr = 0 is the identity, learning on a
planted-partition graph close to the fp32 oracle."""
from fractions import Fraction

import numpy as np
import torch

import oracle
import synth


def _f(bits: int) -> float:
    return float(np.array([bits], np.uint32).view(np.float32)[0])


def _exact(x: float) -> Fraction:
    return Fraction(x)


def _brute_bf16(x: float) -> float:
    """Nearest value whose low 16 bits are zero; ties -> even (bit 16 clear)."""
    u = int(np.array([x], np.float32).view(np.uint32)[0])
    lo = u & 0xFFFF0000
    hi = lo + 0x10000
    a, b = _f(lo), _f(hi)
    if not np.isfinite(b):  # rounding up overflows to inf: exact IEEE behaviour
        if u & 0xFFFF >= 0x8000 and not (u & 0xFFFF == 0x8000 and (lo >> 16) & 1 == 0):
            return b
        return a
    da, db = abs(_exact(x) - _exact(a)), abs(_exact(b) - _exact(x))
    if da < db:
        return a
    if db < da:
        return b
    return a if (lo >> 16) & 1 == 0 else b


def test_round_matches_torch_bfloat16():
    rng = np.random.default_rng(11)
    xs = [rng.normal(0, s, 20000).astype(np.float32) for s in (1e-30, 1e-6, 1e-2, 1.0, 1e3, 1e30)]
    bits = rng.integers(0, 2**32, 200000, dtype=np.uint64).astype(np.uint32)
    rand = bits.view(np.float32)
    rand = rand[np.isfinite(rand)]
    ties = (np.arange(0, 2**16, 7, dtype=np.uint32) << 16 | 0x8000).view(np.float32)
    ties = ties[np.isfinite(ties)]
    specials = np.array([0.0, -0.0, np.inf, -np.inf, 1e-45, -1e-45, 3.4e38, -3.4e38], np.float32)
    x = np.concatenate(xs + [rand, ties, specials])
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    got = oracle.round_bf16(x)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_round_brute_force_bands():
    # every low half-word for a few high half-words: normal, subnormal, negative, near overflow
    for hi in (0x3F80, 0x3F81, 0x0000, 0x0001, 0x8000, 0xBF80, 0x7F7F, 0xC2F6):
        x = ((np.uint32(hi) << np.uint32(16)) | np.arange(0, 2**16, 3, dtype=np.uint32)).view(np.float32)
        got = oracle.round_bf16(x)
        for xi, gi in zip(x[::37], got[::37]):
            assert np.float32(_brute_bf16(float(xi))).view(np.uint32) == np.float32(gi).view(np.uint32), hex(
                int(np.float32(xi).view(np.uint32)))


def test_round_idempotent_and_monotone():
    rng = np.random.default_rng(12)
    x = np.sort(rng.normal(0, 1, 100000).astype(np.float32))
    r = oracle.round_bf16(x)
    assert np.array_equal(oracle.round_bf16(r), r)
    assert (np.diff(r) >= 0).all()
    assert (r.view(np.uint32) & 0xFFFF == 0).all()
    assert np.abs(r - x).max() <= np.abs(x).max() * 2.0**-8


def _graph():
    n = 1500
    u, v = synth.planted_partition_edges(n, 15, 12.0, 1.0, 21)
    off, tgt, test = synth.split_edges(n, u, v, 0.1, 7)
    neg = synth.negative_pairs(n, u, v, len(test), 8)
    return n, off, tgt, test, neg


def test_bf16_epoch_properties():
    n, off, tgt, test, neg = _graph()
    d = 32
    res = {}
    for storage in (0, 1):
        cfg = oracle.Config(dim=d, negatives=5, walk_len=20, window=3, walks_per_node=4, subparts=2,
                            storage=storage)
        V = oracle.init_vertex(n, d, 42)
        if storage:
            V = oracle.round_bf16(V)
        Cm = np.zeros_like(V)
        V0 = V.copy()
        oracle.train_epoch(cfg, off, tgt, V, Cm, 0, 0.0)  # lr = 0: nothing moves
        assert np.array_equal(V, V0) and not Cm.any()
        for ep in range(2):
            oracle.train_epoch(cfg, off, tgt, V, Cm, ep, 0.05)
        if storage:
            assert (V.view(np.uint32) & 0xFFFF == 0).all() and (Cm.view(np.uint32) & 0xFFFF == 0).all()
        res[storage] = (V, Cm, oracle.auc(oracle.score_pairs(V, Cm, test), oracle.score_pairs(V, Cm, neg)))
    assert not np.array_equal(res[0][0], res[1][0])  # the rounding is not a no-op
    assert res[1][2] > 0.9 and abs(res[1][2] - res[0][2]) < 0.02, (res[0][2], res[1][2])
