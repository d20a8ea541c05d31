"""Writes tests/golden/c2_hashes.txt: SHA-256 of the C2 (YouTube-shaped)
walks and of every 2D block of its sample pool, computed by the ORACLE only
(oracle/ + synth/; nothing from the CUDA path).  The GPU parity test compares
the CUDA path's walks and blocks with these hashes ("walks and
samples bit-exact on C2").  Run: python tools/make_golden_c2.py  (~minutes)."""
import hashlib
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402

WALK_EPOCH, POOL_EPOCH, SUBPARTS = 0, 3, 4


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    off, tgt = synth.workload_graph("c2")
    n = len(off) - 1
    lines = ["# C2 youtube-shaped R-MAT (synth.workload_graph('c2')): n=%d nnz=%d" % (n, len(tgt)),
             "# written by tools/make_golden_c2.py from oracle/ only; seed 42, k=40, l=5, w=1, one episode",
             "# walks: sha256 of the u32 [n][41] walk matrix (sentinel 0xFFFFFFFF), epoch %d" % WALK_EPOCH,
             "# block P g vsub: count and sha256 of the (src, dst) u32 pairs, epoch %d, subparts %d"
             % (POOL_EPOCH, SUBPARTS)]
    t = time.time()
    walks = oracle.random_walks(off, tgt, 42, WALK_EPOCH, 0, n, 40)
    lines.append(f"walks {n} {sha(walks)}")
    print(f"walks {time.time() - t:.1f}s", flush=True)
    del walks
    for P in (1, 4):
        t = time.time()
        cfg = oracle.Config(dim=128, negatives=5, walk_len=40, window=5, walks_per_node=1, episodes=1,
                            subparts=SUBPARTS, parts=P, seed=42)
        pairs, boff = oracle.build_episode(cfg, off, tgt, POOL_EPOCH, 0)
        for g in range(P):
            for vs in range(P * SUBPARTS):
                B = vs * P + g
                blk = pairs[int(boff[B]):int(boff[B + 1])]
                lines.append(f"block {P} {g} {vs} {len(blk)} {sha(blk)}")
        print(f"P={P}: {len(pairs)} pairs, {time.time() - t:.1f}s", flush=True)
        del pairs
    with open(os.path.join(ROOT, "tests", "golden", "c2_hashes.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
