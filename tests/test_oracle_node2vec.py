"""Oracle pins for NEXT-1, node2vec second-order walks (Grover & Leskovec 2016,
cited P:355; rejection sampling as in KnightKing, cited P:184): p = q = 1 is
bit-identical to the first-order walk O4; thresholds are exact powers of two
for power-of-two weights; the step distribution after (prev, cur) matches the
closed form alpha(prev, x) * multiplicity(cur, x) / Z."""
import numpy as np
import pytest

import synth


def test_unit_parameters_reduce_to_first_order(orc):
    off, tgt = synth.rmat_graph(800, 5000, 31)
    for w in range(0, 1600, 3):
        a = orc.random_walk(off, tgt, 42, 2, w, 30)
        b = orc.node2vec_walk(off, tgt, 42, 2, w, 30, 1.0, 1.0)
        assert np.array_equal(a, b)


def test_thresholds_exact():
    import oracle as orc
    assert orc.node2vec_thresholds(1.0, 1.0).tolist() == [2**32] * 3
    assert orc.node2vec_thresholds(0.5, 2.0).tolist() == [2**32, 2**31, 2**30]
    assert orc.node2vec_thresholds(4.0, 0.25).tolist() == [2**28, 2**30, 2**32]  # (1/4, 1, 4) / 4


def _two_step_graph():
    # directed: 0 -> {1, 2}; 1 -> {0, 2, 3, 4, 4}; others point back to 1
    src = [0, 0, 1, 1, 1, 1, 1, 2, 3, 4]
    dst = [1, 2, 0, 2, 3, 4, 4, 1, 1, 1]
    return synth.csr_from_directed(5, np.array(src), np.array(dst))


@pytest.mark.parametrize("p,q", [(0.5, 2.0), (2.0, 0.5), (1.0, 0.25), (4.0, 1.0)])
def test_second_step_distribution(orc, p, q):
    off, tgt = _two_step_graph()
    counts = np.zeros(5)
    for r in range(60000):
        path = orc.node2vec_walk(off, tgt, 7, 0, r * 5, 2, p, q)  # start at node 0
        if path[1] == 1:
            counts[path[2]] += 1
    # prev = 0, cur = 1: x=0 returns (1/p); x=2 is adjacent to 0 (1); x=3 and
    # x=4 (multiplicity 2) are farther (1/q)
    w = np.array([1 / p, 0.0, 1.0, 1 / q, 2 / q])
    expect = w / w.sum() * counts.sum()
    nz = expect > 0
    assert counts[~nz].sum() == 0
    chi2 = (((counts[nz] - expect[nz]) ** 2) / expect[nz]).sum()
    assert chi2 < 18.5  # chi^2 with 3 dof, p ~ 3e-4


def test_steps_are_edges_and_deterministic(orc):
    off, tgt = synth.rmat_graph(400, 2500, 33)
    edges = {(u, int(t)) for u in range(400) for t in tgt[int(off[u]):int(off[u + 1])]}
    for w in range(0, 400, 7):
        a = orc.node2vec_walk(off, tgt, 5, 1, w, 25, 0.25, 4.0)
        assert a[0] == w
        for x, y in zip(a[:-1], a[1:]):
            assert (int(x), int(y)) in edges
        assert np.array_equal(a, orc.node2vec_walk(off, tgt, 5, 1, w, 25, 0.25, 4.0))
    # low p (return-happy) revisits the previous node far more often than high p
    def returns(p, q):
        c = 0
        for w in range(400):
            a = orc.node2vec_walk(off, tgt, 5, 1, w, 25, p, q)
            c += sum(int(a[i] == a[i - 2]) for i in range(2, len(a)))
        return c
    assert returns(0.1, 1.0) > 3 * returns(10.0, 1.0)


def test_episode_pool_uses_node2vec(orc):
    off, tgt = synth.rmat_graph(300, 2000, 34)
    cfg = orc.Config(dim=8, negatives=2, walk_len=8, window=2, p=0.5, q=2.0, subparts=1)
    pairs, _ = orc.build_episode(cfg, off, tgt, 0, 0)
    expect = []
    for w in range(300):
        path = orc.node2vec_walk(off, tgt, 42, 0, w, 8, 0.5, 2.0)
        for i in range(len(path)):
            for d in (1, 2):
                if i + d < len(path):
                    expect.append((int(path[i]), int(path[i + d])))
    assert sorted(map(tuple, pairs.tolist())) == sorted(expect)
