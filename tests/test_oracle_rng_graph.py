"""Oracle pins for R1 (Philox), R2 (uniform index), O1 (partitions) and
O3 (alias tables).  Every expected value comes from an external definition
(Random123 KAT, SPEC examples) or from mathematics (closed forms, exact
enumeration), never from the oracle itself."""
import math
from fractions import Fraction

import numpy as np
import pytest

from conftest import golden_lines


# ---------------------------------------------------------------- R1 Philox
def test_philox_known_answers(orc):
    rows = golden_lines("philox4x32_10_kat.txt")
    assert len(rows) == 3
    for row in rows:
        h = [int(x, 16) for x in row.split()]
        out = orc.philox(h[0:4], h[4:6])
        assert [int(x) for x in out] == h[6:10]


def test_philox_counter_sensitivity(orc):
    # flipping any single counter or key bit changes the output (bijection per key)
    base = orc.philox([1, 2, 3, 4], [5, 6])
    for w in range(4):
        ctr = [1, 2, 3, 4]
        ctr[w] ^= 1
        assert not np.array_equal(orc.philox(ctr, [5, 6]), base)
    assert not np.array_equal(orc.philox([1, 2, 3, 4], [5, 7]), base)


# ---------------------------------------------------------------- R2 index
def test_uniform_index_closed_forms(orc):
    rng = np.random.Generator(np.random.PCG64(1))
    for _ in range(200):
        r = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        for j in (0, 1, 5, 17, 32, 40):
            # n = 2^j: floor(r * 2^j / 2^64) = r >> (64 - j)
            assert orc.uniform_index(r, 1 << j) == (r >> (64 - j))
        n = int(rng.integers(1, 2**40))
        # exact floor(r*n/2^64) with Python big ints
        assert orc.uniform_index(r, n) == (r * n) >> 64
    assert orc.uniform_index(0, 12345) == 0
    assert orc.uniform_index(2**64 - 1, 12345) == 12344
    assert orc.uniform_index(2**64 - 1, 1) == 0


# ---------------------------------------------------------------- O1 partitions
def test_partition_examples(orc):
    rows = golden_lines("partition_examples.txt")
    for row in rows:
        if row.startswith("block"):
            lhs, rhs = row[len("block"):].split(":")
            bounds = np.array([int(x) for x in lhs.split()], np.uint64)
            src, dst = [int(x) for x in rhs.split("->")[0].split()]
            exp = [int(x) for x in rhs.split("->")[1].split()]
            assert [orc.part_of(src, bounds), orc.part_of(dst, bounds)] == exp
        else:
            lhs, rhs = row.split("->")
            n, p = [int(x) for x in lhs.split()]
            assert orc.partition_bounds(0, n, p).tolist() == [int(x) for x in rhs.split()]


@pytest.mark.parametrize("n,p", [(1, 1), (7, 3), (1138499, 16), (5, 8), (100, 7), (0, 2)])
def test_partition_cover(orc, n, p):
    b = orc.partition_bounds(0, n, p).astype(np.int64)
    sizes = np.diff(b)
    assert b[0] == 0 and b[-1] == n
    assert (sizes >= 0).all() and sizes.max() - sizes.min() <= 1
    # remainder goes to the earlier parts
    assert (np.diff(sizes) <= 0).all()
    # part_of agrees with an independent range search
    for v in np.random.default_rng(0).integers(0, max(n, 1), 50):
        if n:
            assert orc.part_of(int(v), b.astype(np.uint64)) == int(np.searchsorted(b, v, side="right") - 1)


# ---------------------------------------------------------------- O3 alias
def test_weight075_exact_powers(orc):
    for d, w in [(0, 0.0), (1, 1.0), (16, 8.0), (81, 27.0), (256, 64.0), (10000, 1000.0)]:
        assert orc.weight075(d) == w
    for d in [2, 3, 7, 1000, 123456, 10**7]:
        assert math.isclose(orc.weight075(d), d ** 0.75, rel_tol=4e-16)


def _implied_distribution(thr, al):
    """Exact output distribution of (column uniform, coin x2 uniform u32):
    P(i) = (1/n) sum_c [c == i] thr_c/2^32 + [alias_c == i] (1 - thr_c/2^32)."""
    n = len(thr)
    P = [Fraction(0)] * n
    for c in range(n):
        keep = Fraction(int(thr[c]), 2**32)
        P[c] += keep / n
        P[int(al[c])] += (1 - keep) / n
    return P


def test_alias_examples(orc):
    for row in golden_lines("alias_examples.txt"):
        lhs, rhs = row.split("->")
        deg = [int(x) for x in lhs.split()]
        expect = [float(x) for x in rhs.split()]
        thr, al = orc.alias_build(deg)
        P = _implied_distribution(thr, al)
        for p, e in zip(P, expect):
            assert abs(float(p) - e) <= len(deg) * 2.0**-32


def test_alias_equal_degrees_uniform_exact(orc):
    thr, al = orc.alias_build([5] * 17)
    assert (thr == 0xFFFFFFFF).all() and (al == np.arange(17)).all()


def test_alias_all_zero_uniform_fallback(orc):
    thr, al = orc.alias_build([0, 0, 0])
    P = _implied_distribution(thr, al)
    for p in P:
        assert abs(float(p) - 1 / 3) <= 3 * 2.0**-32


@pytest.mark.parametrize("seed", range(6))
def test_alias_integer_invariant_and_distribution(orc, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300))
    deg = rng.integers(0, 2000, n) * (rng.random(n) < 0.8)
    deg[rng.integers(0, n)] = rng.integers(1, 5000)
    num, al, W = orc.alias_masses(deg)
    q = [0 if d == 0 else math.floor(orc.weight075(int(d)) * 2**20 + 0.5) for d in deg]
    assert W == sum(q)
    # exact reconstruction: num_i + sum_{c: alias_c = i, c != i} (W - num_c) == q_i * n
    recon = [int(x) for x in num]
    for c in range(n):
        if int(al[c]) != c:
            recon[int(al[c])] += W - int(num[c])
        else:
            assert int(num[c]) == W
    assert recon == [qi * n for qi in q]
    # implied sampling distribution within n * 2^-32 of q / sum(q)
    thr, al2 = orc.alias_build(deg)
    assert (al2 == al).all()
    P = _implied_distribution(thr, al2)
    for p, qi in zip(P, q):
        assert abs(float(p) - qi / W) <= n * 2.0**-32 + 1e-15


def test_alias_pick_branches(orc):
    thr = np.array([0x80000000, 0xFFFFFFFF, 0], np.uint32)
    al = np.array([1, 1, 0], np.uint32)
    n = 3
    for col in range(n):
        r64 = (col * 2**64 + n - 1) // n       # smallest r64 with floor(r64*n/2^64) == col
        x0, x1 = r64 & 0xFFFFFFFF, r64 >> 32
        t = int(thr[col])
        if t > 0:
            assert orc.alias_pick(thr, al, x0, x1, t - 1) == col      # coin below threshold: keep
        assert orc.alias_pick(thr, al, x0, x1, min(t, 2**32 - 1)) == (col if t == 2**32 - 1 else int(al[col]))


def test_alias_sampling_chi_square(orc):
    deg = np.array([1, 16, 3, 0, 40, 7], np.uint64)
    thr, al = orc.alias_build(deg)
    w = np.array([orc.weight075(int(d)) for d in deg])
    p = w / w.sum()
    draws = 60000
    rng = np.random.default_rng(3)
    x = rng.integers(0, 2**32, size=(draws, 3), dtype=np.uint64)
    cnt = np.zeros(len(deg))
    for a, b, c in x.tolist():
        cnt[orc.alias_pick(thr, al, a, b, c)] += 1
    nz = p > 0
    assert cnt[~nz].sum() == 0
    chi2 = (((cnt[nz] - draws * p[nz]) ** 2) / (draws * p[nz])).sum()
    assert chi2 < 20.5  # chi^2_4, p = 0.0004
