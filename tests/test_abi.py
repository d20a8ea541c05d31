"""The C-ABI library loads without a GPU and exports every symbol include/ne.h
declares; host-only entry points (plan, partitions) and argument validation
work on the CPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ne.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ne_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2005_13789_b200 import ne
    lib = ctypes.CDLL(ne.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(ne.EXPORTED)
    assert ne.ne_version() == 2


def test_host_plan_matches_oracle_plan(orc):
    from paper_2005_13789_b200 import ne
    for P in (1, 2, 3, 8):
        for k in (1, 4):
            for r in range(P + 1):
                for t in range(k):
                    for g in range(P):
                        assert ne.ne_plan_vsub(P, k, r, t, g) == orc.plan_vsub(P, k, r, t, g)
    assert ne.ne_plan_vsub(0, 1, 0, 0, 0) == -1


def test_host_partitions_match_oracle(orc):
    from paper_2005_13789_b200 import ne
    for n, p in [(8, 2), (9, 2), (1138499, 16), (5, 8)]:
        assert np.array_equal(ne.ne_partition_bounds(n, p), orc.partition_bounds(0, n, p))


def test_create_validates_config_without_gpu():
    from paper_2005_13789_b200 import ne
    with pytest.raises(ne.NEError, match="NE_EINVAL: dim=130"):
        ne.ne_create(ne.ne_config(130, 5, 40, 5, 1, 1, 4, 0, 0, 0, 1.0, 1.0, 0, 0, 0, 0, 42), 0)
    with pytest.raises(ne.NEError, match="NE_EINVAL: negatives=9"):
        ne.ne_create(ne.ne_config(128, 9, 40, 5, 1, 1, 4, 0, 0, 0, 1.0, 1.0, 0, 0, 0, 0, 42), 0)
    with pytest.raises(ne.NEError, match="NE_EINVAL: window=6"):
        ne.ne_create(ne.ne_config(128, 5, 5, 6, 1, 1, 4, 0, 0, 0, 1.0, 1.0, 0, 0, 0, 0, 42), 0)


def test_create_validates_node2vec_and_writeback():
    from paper_2005_13789_b200 import ne
    with pytest.raises(ne.NEError, match="NE_EINVAL: node2vec p=-1"):
        ne.ne_create(ne.ne_config(128, 5, 40, 5, 1, 1, 4, 0, 0, 0, -1.0, 1.0, 0, 0, 0, 0, 42), 0)
    with pytest.raises(ne.NEError, match="NE_EINVAL: writeback=7"):
        ne.ne_create(ne.ne_config(128, 5, 40, 5, 1, 1, 4, 0, 0, 7, 1.0, 1.0, 0, 0, 0, 0, 42), 0)
    with pytest.raises(ne.NEError, match="NE_EINVAL: episodes=0"):
        ne.ne_create(ne.ne_config(128, 5, 40, 5, 1, 0, 4, 0, 0, 0, 1.0, 1.0, 0, 0, 0, 0, 42), 0)


def test_create_validates_update_rule():
    from paper_2005_13789_b200 import ne
    with pytest.raises(ne.NEError, match="NE_EINVAL: update_rule=2"):
        ne.ne_create(ne.ne_config(128, 5, 40, 5, 1, 1, 4, 0, 0, 0, 1.0, 1.0, 2, 0, 0, 0, 42), 0)
    with pytest.raises(ne.NEError, match="NE_EINVAL: staging=3"):
        ne.ne_create(ne.ne_config(128, 5, 40, 5, 1, 1, 4, 0, 0, 0, 1.0, 1.0, 0, 3, 0, 0, 42), 0)


def test_create_validates_storage():
    from paper_2005_13789_b200 import ne
    with pytest.raises(ne.NEError, match="NE_EINVAL: storage=2"):
        ne.ne_create(ne.ne_config(128, 5, 40, 5, 1, 1, 4, 0, 0, 0, 1.0, 1.0, 0, 0, 2, 0, 42), 0)
    with pytest.raises(ne.NEError, match="NE_EINVAL: transport=2"):
        ne.ne_create(ne.ne_config(128, 5, 40, 5, 1, 1, 4, 0, 0, 0, 1.0, 1.0, 0, 0, 0, 2, 42), 0)



def test_two_level_plan_matches_oracle(orc):
    """NEXT-3: the library's two-level plan and ring hops (host code, no
    device) against the oracle's or_plan_vsub2."""
    from paper_2005_13789_b200 import ne
    for P, G in [(1, 1), (2, 1), (2, 2), (4, 2), (6, 3), (8, 2), (8, 4), (8, 8)]:
        for k in (1, 3):
            for rho in range(P):
                for t in range(k):
                    for g in range(P):
                        s = ne.ne_plan_vsub2(P, G, k, rho, t, g)
                        assert s == orc.plan_vsub2(P, G, k, rho, t, g)
                        dest, src = ne.ne_ring_peers(P, G, rho, g)
                        # the sub-part moves to dest, which trains it next round (home after the last)
                        assert ne.ne_plan_vsub2(P, G, k, rho + 1, t, dest) == s
                        assert ne.ne_ring_peers(P, G, rho, src)[0] == g
    assert ne.ne_plan_vsub2(6, 4, 1, 0, 0, 0) == -1
