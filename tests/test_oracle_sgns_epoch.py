"""Oracle pins for O9 (init), O10 (SGNS update), O7/O11 (epoch plan) and
O12 (AUC).  Expected values: SPEC's worked examples, finite differences of the
loss, exact special cases (eta = 0, zero rows), composition, orthogonality
(block order within a step is immaterial) and a learning pin (held-out AUC on a
planted-partition graph)."""
import math

import numpy as np
import pytest

import synth
from conftest import golden_kv, golden_lines


def _cfg(orc, **kw):
    base = dict(dim=16, negatives=5, walk_len=10, window=3, walks_per_node=1, episodes=1,
                subparts=2, parts=1, seed=42)
    base.update(kw)
    return orc.Config(**base)


# ---------------------------------------------------------------- O10
def test_sigmoid_examples_and_clamp(orc):
    g = golden_kv("sgns_worked_example.txt")
    tol = float(g["tolerance"])
    assert orc.sigmoid(0.0) == float(g["sigma_0"])
    assert abs(orc.sigmoid(1.0) - float(g["sigma_1"])) < tol
    assert orc.sigmoid(40.0) == orc.sigmoid(30.0) and orc.sigmoid(-40.0) == orc.sigmoid(-30.0)
    assert 0.0 < orc.sigmoid(-1e9) < orc.sigmoid(1e9) < 1.0


def test_sigmoid_clamp_closed_form(orc):
    """The +-30 clamp (reading D11) pinned by closed-form values: sigma(10) and
    sigma(-10) unclamped, sigma strictly increasing up to 30 and constant beyond,
    and the loss of one update (lr = 0, so rows stay put) at |v.c| = 25 and 40."""
    g = golden_kv("sigma_clamp.txt")
    assert abs(orc.sigmoid(10.0) - float(g["sigma_10"])) <= 1e-16
    assert abs(orc.sigmoid(-10.0) - float(g["sigma_minus_10"])) <= 1e-20
    b = float(g["clamp"])
    assert orc.sigmoid(b - 1) < orc.sigmoid(b - 0.5) < orc.sigmoid(b)
    assert orc.sigmoid(-b) < orc.sigmoid(-b + 0.5) < orc.sigmoid(-b + 1)
    assert orc.sigmoid(b + 1) == orc.sigmoid(b) == orc.sigmoid(1e6)
    assert orc.sigmoid(-b - 1) == orc.sigmoid(-b) == orc.sigmoid(-1e6)
    # -log(1 - s) at s = sigma(30) = 1 - 9.4e-14 loses ~1e-3 of 1 - s to cancellation
    # (eps / 9.4e-14); a +-6 clamp would give 6.0025 and no clamp 40
    for x, label, key, tol in ((-25.0, 1, "loss_pos_at_minus_25", 1e-12), (-40.0, 1, "loss_pos_at_minus_40", 1e-12),
                               (40.0, 0, "loss_neg_at_40", 2e-3)):
        v = np.array([x / 4] * 4, np.float32)
        c = np.ones(4, np.float32)
        loss = orc.sgns_step(v, c, label, 0.0)
        assert abs(loss - float(g[key])) <= tol, (x, label, loss)


def test_worked_update(orc):
    g = golden_kv("sgns_worked_example.txt")
    tol = float(g["tolerance"])
    v = np.array(g["update_v"].split(), np.float32)
    c = np.array(g["update_c"].split(), np.float32)
    gv, gc, _ = orc.sgns_grad(v, c, int(g["update_label"]))
    # dL/dv = g * c with c = [1, 0]
    assert abs(gv[0] - float(g["update_g"])) < tol
    orc.sgns_step(v, c, int(g["update_label"]), float(g["update_eta"]))
    assert np.allclose(v, np.array(g["update_v_out"].split(), np.float32), atol=tol, rtol=0)
    assert np.allclose(c, np.array(g["update_c_out"].split(), np.float32), atol=tol, rtol=0)


def test_zero_rows_unchanged(orc):
    for label in (0, 1):
        v = np.zeros(8, np.float32)
        c = np.zeros(8, np.float32)
        loss = orc.sgns_step(v, c, label, 0.5)
        assert not v.any() and not c.any()
        assert math.isclose(loss, math.log(2.0), rel_tol=1e-15)


def test_gradient_matches_finite_differences(orc):
    # 100 random instances, d <= 16, rel err <= 1e-4 in double
    rng = np.random.default_rng(0)

    def loss(v, c, y):
        return orc.sgns_grad(v, c, y)[2]

    for _ in range(100):
        d = int(rng.integers(1, 17))
        v = rng.normal(0, 0.7, d)
        c = rng.normal(0, 0.7, d)
        y = int(rng.integers(0, 2))
        gv, gc, _ = orc.sgns_grad(v, c, y)
        h = 1e-5
        fv = np.zeros(d)
        fc = np.zeros(d)
        for i in range(d):
            e = np.zeros(d)
            e[i] = h
            fv[i] = (loss(v + e, c, y) - loss(v - e, c, y)) / (2 * h)
            fc[i] = (loss(v, c + e, y) - loss(v, c - e, y)) / (2 * h)
        num = np.linalg.norm(np.concatenate([gv - fv, gc - fc]))
        den = max(np.linalg.norm(np.concatenate([fv, fc])), 1e-12)
        assert num / den <= 1e-4


def test_positive_updates_increase_score(orc):
    # 2-node graph, m = 0, repeated positive updates increase sigma(v.c)
    V = orc.init_vertex(2, 4, 3)
    Cm = np.full((2, 4), 0.01, np.float32)
    prev = -1.0
    for _ in range(200):
        orc.train_sample(V, Cm, 0, 1, np.zeros(0, np.uint32), 0.1)
        s = orc.score_pairs(V, Cm, np.array([[0, 1]], np.uint32))[0]
        assert s > prev
        prev = s


def test_sample_is_composition_of_steps(orc):
    # K = 0 is one update; K > 0 applies the 1+K updates in order, a
    # repeated context id seeing its earlier update (reading D2)
    rng = np.random.default_rng(1)
    d = 12
    V = rng.normal(0, 0.3, (5, d)).astype(np.float32)
    Cm = rng.normal(0, 0.3, (5, d)).astype(np.float32)
    for negs in ([], [3], [2, 4, 2], [1, 1, 3, 1]):
        V1, C1 = V.copy(), Cm.copy()
        l1 = orc.train_sample(V1, C1, 0, 1, np.array(negs, np.uint32), 0.05)
        V2, C2 = V.copy(), Cm.copy()
        l2 = orc.sgns_step(V2[0], C2[1], 1, 0.05)
        for j in negs:
            row = C2[j].copy()
            l2 += orc.sgns_step(V2[0], row, 0, 0.05)
            C2[j] = row
        assert np.array_equal(V1, V2) and np.array_equal(C1, C2)
        assert l1 == l2


# ---------------------------------------------------------------- O9
def test_init_range_and_grid(orc):
    for d in (1, 16, 96, 100, 128):
        V = orc.init_vertex(300, d, 42)
        assert (np.abs(V) <= 0.5 / d).all()
        if d & (d - 1) == 0:
            # d a power of two: the division is exact, so (V*d + 0.5) * 2^24 is
            # an integer in [0, 2^24) -- a 24-bit uniform grid
            k = (V.astype(np.float64) * d + 0.5) * 2**24
            assert np.array_equal(k, np.round(k)) and k.min() >= 0 and k.max() < 2**24
    V = orc.init_vertex(20000, 8, 42)
    u = (V.reshape(-1).astype(np.float64) * 8 + 0.5)
    # uniform on [0,1): mean 1/2, variance 1/12, KS distance small
    assert abs(u.mean() - 0.5) < 0.005 and abs(u.var() - 1 / 12) < 0.002
    s = np.sort(u)
    assert np.abs(s - (np.arange(len(s)) + 0.5) / len(s)).max() < 0.01
    # rows start where they say they start
    assert np.array_equal(orc.init_vertex(10, 8, 42, row_begin=5), orc.init_vertex(15, 8, 42)[5:])
    assert not np.array_equal(orc.init_vertex(10, 8, 42), orc.init_vertex(10, 8, 43))


# ---------------------------------------------------------------- O7 / O11
def test_eta_zero_epoch_is_identity(orc):
    off, tgt = synth.rmat_graph(200, 1000, 3)
    cfg = _cfg(orc)
    V = orc.init_vertex(200, 16, 42)
    V0 = V.copy()
    Cm = np.zeros_like(V)
    ns, loss = orc.train_epoch(cfg, off, tgt, V, Cm, 0, 0.0)
    assert np.array_equal(V, V0) and not Cm.any()
    # C = 0 => every score is 1/2 => loss = (1 + K) log 2 per sample
    assert math.isclose(loss, ns * 6 * math.log(2.0), rel_tol=1e-12)
    pairs, _ = orc.build_episode(cfg, off, tgt, 0, 0)
    assert ns == len(pairs)


@pytest.mark.parametrize("P,k", [(2, 1), (2, 2), (3, 2), (4, 1)])
def test_block_order_within_step_is_immaterial(orc, P, k):
    # P:89 orthogonality: the blocks of one (round, slot) step touch disjoint
    # rows, so replaying them in reverse gives bit-identical embeddings
    off, tgt = synth.rmat_graph(240, 2000, 12)
    cfg = _cfg(orc, parts=P, subparts=k)
    V = orc.init_vertex(240, 16, 42)
    Cm = np.zeros_like(V)
    V2, C2 = V.copy(), Cm.copy()
    orc.train_epoch(cfg, off, tgt, V, Cm, 0, 0.05)
    orc.train_epoch(cfg, off, tgt, V2, C2, 0, 0.05, reverse_within_step=True)
    assert np.array_equal(V, V2) and np.array_equal(Cm, C2)


def test_plan_examples(orc):
    # S:307-308 blocks_for_step (N,G,k) = (1,2,1): step 0 -> worker0:(0,0),
    # worker1:(1,1); step 1 -> worker0:(1,0), worker1:(0,1)
    assert [(orc.plan_vsub(2, 1, 0, 0, g), g) for g in range(2)] == [(0, 0), (1, 1)]
    assert [(orc.plan_vsub(2, 1, 1, 0, g), g) for g in range(2)] == [(1, 0), (0, 1)]
    # Fig. 4, two GPUs, k = 2: after the first exchange GPU1
    # (g=0) holds block 2_1 (vertex part 1, slot 0) and GPU2 holds 1_1
    assert orc.plan_vsub(2, 2, 1, 0, 0) == 1 * 2 + 0
    assert orc.plan_vsub(2, 2, 1, 0, 1) == 0 * 2 + 0


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("k", [1, 2, 4])
def test_plan_latin_square_and_ring(orc, P, k):
    seen = set()
    for r in range(P):
        for t in range(k):
            step = [orc.plan_vsub(P, k, r, t, g) for g in range(P)]
            assert len(set(step)) == P                       # (a) orthogonal per step
            for g, s in enumerate(step):
                seen.add((s, g))
                assert s % k == t                            # slot t of some part
                if r + 1 < P:                                # ring: g receives from g-1
                    assert orc.plan_vsub(P, k, r + 1, t, (g + 1) % P) == s
            # round 0 trains the GPU's own (home) vertex part
            if r == 0:
                assert step == [g * k + t for g in range(P)]
    assert seen == {(s, g) for s in range(P * k) for g in range(P)}   # (c) coverage


@pytest.mark.parametrize("P,k,E", [(2, 2, 2), (3, 1, 1)])
def test_epoch_equals_replay_of_pool(orc, P, k, E):
    # the epoch = ring-order replay of the pool's blocks with O8 negatives
    off, tgt = synth.rmat_graph(150, 800, 2)
    cfg = _cfg(orc, parts=P, subparts=k, episodes=E)
    V = orc.init_vertex(150, 16, 42)
    Cm = np.zeros_like(V)
    V2, C2 = V.copy(), Cm.copy()
    orc.train_epoch(cfg, off, tgt, V, Cm, 3, 0.05)
    thr, al = orc.build_alias_tables(cfg, off)
    pb = orc.partition_bounds(0, 150, P).astype(np.int64)
    for e in range(E):
        pairs, boff = orc.build_episode(cfg, off, tgt, 3, e)
        for r in range(P):
            for t in range(k):
                for g in range(P):
                    B = (((g - r) % P) * k + t) * P + g   # ring: part (g - r) mod P
                    for p in range(int(boff[B + 1] - boff[B])):
                        src, dst = pairs[int(boff[B]) + p]
                        negs = orc.negatives(cfg, thr, al, int(pb[g]), int(pb[g + 1] - pb[g]), 3, e, B, p)
                        orc.train_sample(V2, C2, int(src), int(dst), negs, 0.05)
    assert np.array_equal(V, V2) and np.array_equal(Cm, C2)


def test_link_prediction_learns(orc):
    # the method's purpose: held-out edges of a community
    # graph score above random non-edges after a few epochs
    n = 2000
    u, v = synth.planted_partition_edges(n, 20, 12.0, 1.0, 17)
    off, tgt, test = synth.split_edges(n, u, v, 0.1, 7)
    neg = synth.negative_pairs(n, u, v, len(test), 8)
    cfg = _cfg(orc, dim=32, walk_len=20, window=3, walks_per_node=4, subparts=1)
    V = orc.init_vertex(n, 32, 42)
    Cm = np.zeros_like(V)
    a0 = orc.auc(orc.score_pairs(V, Cm, test), orc.score_pairs(V, Cm, neg))
    assert a0 == 0.5   # C = 0: every score is 1/2
    for ep in range(2):
        orc.train_epoch(cfg, off, tgt, V, Cm, ep, 0.05)
    a = orc.auc(orc.score_pairs(V, Cm, test), orc.score_pairs(V, Cm, neg))
    assert a > 0.9


# ---------------------------------------------------------------- O12
def test_auc_examples(orc):
    for row in golden_lines("auc_examples.txt"):
        lhs, rhs = row.split("->")
        pos, neg = lhs.split("|")
        pos = [float(x) for x in pos.split()]
        neg = [float(x) for x in neg.split()]
        assert orc.auc(pos, neg) == float(rhs)


def test_auc_matches_bruteforce_with_ties(orc):
    rng = np.random.default_rng(4)
    for _ in range(200):
        a = rng.integers(0, 20, int(rng.integers(1, 60))) / 10.0
        b = rng.integers(0, 20, int(rng.integers(1, 60))) / 10.0
        assert orc.auc(a, b) == orc.auc_bruteforce(a, b)
        assert orc.auc(a, a) == 0.5
        assert orc.auc(np.exp(a), np.exp(b)) == orc.auc(a, b)


# ---------------------------------------------------------------- NEXT-3 two-level ring
@pytest.mark.parametrize("P", [1, 2, 3, 4, 6, 8])
@pytest.mark.parametrize("k", [1, 2, 4])
def test_two_level_plan_reduces_to_single_ring(orc, P, k):
    # one group (one node) or one rank per group: both are the single ring
    for rho in range(P):
        for t in range(k):
            for g in range(P):
                s = orc.plan_vsub(P, k, rho, t, g)
                assert orc.plan_vsub2(P, 1, k, rho, t, g) == s
                assert orc.plan_vsub2(P, P, k, rho, t, g) == s


@pytest.mark.parametrize("P,G", [(4, 2), (6, 2), (6, 3), (8, 2), (8, 4), (12, 3)])
@pytest.mark.parametrize("k", [1, 2, 4])
def test_two_level_plan_invariants(orc, P, G, k):
    """SPEC build_schedule invariants, brute force: (a) per step no
    sub-part on two ranks; (c) every (sub-part, context part) exactly once;
    within a macro-round sub-parts rotate along the group's ring, between
    macro-rounds the group's sub-parts move to the next group;
    the first macro-round trains the group's own vertex parts ("all GPUs
    from Node0 will first train on half of the vertex embeddings")."""
    L = P // G
    seen = set()
    for rho in range(P):
        R, r = divmod(rho, L)
        for t in range(k):
            step = [orc.plan_vsub2(P, G, k, rho, t, g) for g in range(P)]
            assert len(set(step)) == P
            for g, s in enumerate(step):
                a, j = divmod(g, L)
                seen.add((s, g))
                assert s % k == t
                part = s // k
                assert part // L == (a - R) % G          # the group holds group (a - R)'s parts
                if R == 0:
                    assert part // L == a                # first macro-round: its own parts
                nxt = a * L + (j + 1) % L if r < L - 1 else ((a + 1) % G) * L + (j + 1) % L
                if rho + 1 < P:
                    assert orc.plan_vsub2(P, G, k, rho + 1, t, nxt) == s
                else:                                    # the final hop returns it home
                    assert part == nxt
    assert seen == {(s, g) for s in range(P * k) for g in range(P)}


def test_two_level_epoch_equals_replay(orc):
    # the oracle's epoch with groups = ordered replay of the two-level plan;
    # and the plan matters: the single ring gives a different result
    P, G, k = 4, 2, 2
    off, tgt = synth.rmat_graph(160, 900, 6)
    cfg = _cfg(orc, parts=P, subparts=k, groups=G)
    V = orc.init_vertex(160, 16, 42)
    Cm = np.zeros_like(V)
    V2, C2, V3, C3 = V.copy(), Cm.copy(), V.copy(), Cm.copy()
    orc.train_epoch(cfg, off, tgt, V, Cm, 1, 0.05)
    thr, al = orc.build_alias_tables(cfg, off)
    pb = orc.partition_bounds(0, 160, P).astype(np.int64)
    pairs, boff = orc.build_episode(cfg, off, tgt, 1, 0)
    L = P // G
    for rho in range(P):
        R, r = divmod(rho, L)
        for t in range(k):
            for g in range(P):
                a, j = divmod(g, L)
                B = ((((a - R) % G) * L + (j - r) % L) * k + t) * P + g
                for p in range(int(boff[B + 1] - boff[B])):
                    src, dst = pairs[int(boff[B]) + p]
                    negs = orc.negatives(cfg, thr, al, int(pb[g]), int(pb[g + 1] - pb[g]), 1, 0, B, p)
                    orc.train_sample(V2, C2, int(src), int(dst), negs, 0.05)
    assert np.array_equal(V, V2) and np.array_equal(Cm, C2)
    orc.train_epoch(_cfg(orc, parts=P, subparts=k), off, tgt, V3, C3, 1, 0.05)
    assert not np.array_equal(V, V3)


def test_windowed_plan_order(orc):
    """NEXT-2 staged ring (reading D18): with window_slots = w the epoch trains
    the slots in windows of w, every window through all P rounds before the
    next; w = k (or 0) is the plain plan, and w < k is the same set of blocks
    in that order (replay)."""
    P, k, w = 2, 4, 2
    off, tgt = synth.rmat_graph(150, 900, 12)
    V = orc.init_vertex(150, 16, 42)
    Cm = np.zeros_like(V)
    ref = [(V.copy(), Cm.copy()) for _ in range(3)]
    orc.train_epoch(_cfg(orc, parts=P, subparts=k), off, tgt, *ref[0], 0, 0.05)
    orc.train_epoch(_cfg(orc, parts=P, subparts=k, window_slots=k), off, tgt, *ref[1], 0, 0.05)
    assert np.array_equal(ref[0][0], ref[1][0]) and np.array_equal(ref[0][1], ref[1][1])
    cfg = _cfg(orc, parts=P, subparts=k, window_slots=w)
    orc.train_epoch(cfg, off, tgt, *ref[2], 0, 0.05)
    assert not np.array_equal(ref[2][0], ref[0][0])
    thr, al = orc.build_alias_tables(cfg, off)
    pb = orc.partition_bounds(0, 150, P).astype(np.int64)
    pairs, boff = orc.build_episode(cfg, off, tgt, 0, 0)
    V2, C2 = V.copy(), Cm.copy()
    for t0 in range(0, k, w):
        for r in range(P):
            for t in range(t0, t0 + w):
                for g in range(P):
                    B = (((g - r) % P) * k + t) * P + g
                    for p in range(int(boff[B + 1] - boff[B])):
                        src, dst = pairs[int(boff[B]) + p]
                        negs = orc.negatives(cfg, thr, al, int(pb[g]), int(pb[g + 1] - pb[g]), 0, 0, B, p)
                        orc.train_sample(V2, C2, int(src), int(dst), negs, 0.05)
    assert np.array_equal(ref[2][0], V2) and np.array_equal(ref[2][1], C2)
