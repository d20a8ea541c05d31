"""NEXT-4 shared-negative mini-batch rule (update_rule = 2, reading D17) on the
tcgen05 tensor-core kernel (kernels_sgns_batch.cu) against the oracle variant
(or_train_batch): the deterministic mode (one CTA, batches in canonical order)
element-wise within the tf32 bound below, and the Hogwild mode by held-out
link-prediction AUC within 0.01."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

# tf32 products: each factor keeps 10 explicit mantissa bits (relative rounding
# <= 2^-11), so every gradient entry is off by up to ~2^-10 of its magnitude,
# and SGD compounds it over the epochs.  The bar: relative Frobenius error of
# each matrix <= 1e-3 (~2^-10), max-abs <= 2^-7 of the matrix's largest
# entry (measured 2^-8); a short run at a small lr (the ragged test) stays
# within 2e-5.
TOL_REL = 1e-3
TOL_ABS = 2e-5


def _engine(**kw):
    from paper_2005_13789_b200.engine import Engine
    base = dict(dim=128, negatives=32, walk_len=10, window=3, walks_per_node=1, episodes=1, subparts=2,
                deterministic=True, seed=42, device=0, update_rule=2)
    base.update(kw)
    return Engine(**base)


def _ocfg(**kw):
    base = dict(dim=128, negatives=32, walk_len=10, window=3, walks_per_node=1, episodes=1, subparts=2,
                parts=1, seed=42, update_rule=2, batch=128)
    base.update(kw)
    return oracle.Config(**base)


@pytest.mark.parametrize("kp,epochs", [(32, 2)])
def test_batch_rule_deterministic_matches_oracle(kp, epochs):
    off, tgt = synth.rmat_graph(2500, 15000, 21)
    n = len(off) - 1
    eng = _engine(negatives=kp)
    eng.load_graph(off, tgt)
    V = oracle.init_vertex(n, 128, 42)
    Cm = np.zeros_like(V)
    cfg = _ocfg(negatives=kp)
    for ep in range(epochs):
        st = eng.train_epoch(ep, 0.025)
        ns, loss = oracle.train_epoch(cfg, off, tgt, V, Cm, ep, 0.025)
        assert st["samples"] == ns
        # the loss sums sigma of tf32 logits: each logit is off by up to 2^-10 of its term magnitudes
        assert abs(st["loss_sum"] - loss) <= 2e-3 * abs(loss), (st["loss_sum"], loss)
    Vg, Cg = eng.embeddings(0), eng.embeddings(1)
    eng.close()
    for got, ref in ((Vg, V), (Cg, Cm)):
        err = float(np.abs(got - ref).max())
        rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        print(f"K'={kp}: max-abs {err:.3e}, relative Frobenius {rel:.3e}")
        assert err <= 2.0 ** -7 * float(np.abs(ref).max()) and rel <= TOL_REL, (err, rel)


def test_batch_rule_ragged_and_tiny_blocks():
    """Blocks smaller than one batch and ragged last batches (padding rows)."""
    # (a small lr: on a 300-node graph a batch sums the gradients of many
    # repeated hub rows, and lr = 0.05 makes the exact rule itself diverge)
    off, tgt = synth.rmat_graph(300, 1200, 22)
    n = len(off) - 1
    eng = _engine(subparts=3, walk_len=4, window=2)
    eng.load_graph(off, tgt)
    st = eng.train_epoch(0, 0.005)
    V = oracle.init_vertex(n, 128, 42)
    Cm = np.zeros_like(V)
    ns, _ = oracle.train_epoch(_ocfg(subparts=3, walk_len=4, window=2), off, tgt, V, Cm, 0, 0.005)
    assert st["samples"] == ns and ns % 128 != 0
    assert np.abs(eng.embeddings(0) - V).max() <= TOL_ABS
    assert np.abs(eng.embeddings(1) - Cm).max() <= TOL_ABS
    eng.close()


def test_batch_rule_hogwild_auc():
    n = 2000
    u, v = synth.planted_partition_edges(n, 20, 12.0, 1.0, 17)
    off, tgt, test = synth.split_edges(n, u, v, 0.1, 7)
    neg = synth.negative_pairs(n, u, v, len(test), 8)
    kw = dict(walk_len=20, window=3, walks_per_node=4, subparts=1)
    cfg = _ocfg(**kw)
    V = oracle.init_vertex(n, 128, 42)
    Cm = np.zeros_like(V)
    for ep in range(2):
        oracle.train_epoch(cfg, off, tgt, V, Cm, ep, 0.05)
    a_ref = oracle.auc(oracle.score_pairs(V, Cm, test), oracle.score_pairs(V, Cm, neg))
    aucs = []
    for run in range(2):
        eng = _engine(deterministic=False, **kw)
        eng.load_graph(off, tgt)
        for ep in range(2):
            eng.train_epoch(ep, 0.05)
        Vg, Cg = eng.embeddings(0), eng.embeddings(1)
        aucs.append(oracle.auc(oracle.score_pairs(Vg, Cg, test), oracle.score_pairs(Vg, Cg, neg)))
        eng.close()
    print("batch-rule AUC: oracle", a_ref, "gpu", aucs)
    assert a_ref > 0.8 and all(abs(a - a_ref) <= 0.01 for a in aucs), (a_ref, aucs)


def test_batch_rule_rejects_unsupported_shapes():
    from paper_2005_13789_b200 import ne
    for kw in (dict(dim=96), dict(negatives=5), dict(negatives=64)):
        with pytest.raises(ne.NEError, match="update_rule=2"):
            _engine(**kw)


def test_umma_products_match_numpy():
    """The batch kernel's three tcgen05 tf32 products (tiles, descriptors, TMEM
    read-back) against fp64 numpy products of the same inputs: tf32 keeps 10
    mantissa bits of each factor, so |error| <= 2^-10 * sum |a_k b_k| bounds
    each entry."""
    from paper_2005_13789_b200 import ne
    rng = np.random.default_rng(3)
    V = rng.normal(0, 1, (128, 128)).astype(np.float32)
    N = rng.normal(0, 1, (32, 128)).astype(np.float32)
    G = rng.normal(0, 1, (128, 32)).astype(np.float32)
    S, dV, dNt = ne.ne_umma_products(V, N, G)
    V64, N64, G64 = V.astype(np.float64), N.astype(np.float64), G.astype(np.float64)
    for got, ref, bound in ((S, V64 @ N64.T, np.abs(V64) @ np.abs(N64.T)),
                            (dV, G64 @ N64, np.abs(G64) @ np.abs(N64)),
                            (dNt, V64.T @ G64, np.abs(V64.T) @ np.abs(G64))):
        err = np.abs(got - ref)
        assert (err <= 2.0 ** -10 * bound + 1e-5).all(), float((err / (bound + 1e-30)).max())
