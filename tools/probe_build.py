"""Walk + pool build of rank 0 of P (layout-only context, one GPU): the
per-rank build cost of the multi-GPU path, for ncu launch lists."""
import sys, time
sys.path.insert(0, ".")
import synth
from paper_2005_13789_b200.engine import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 4
off, tgt = synth.workload_graph(name, device="cuda")
w = synth.CONFIGS[name]
eng = Engine(dim=w.dim, episodes=w.episodes, rank=0, world=P, p=w.p, q=w.q)
eng.load_graph(off, tgt)
for ep in range(3):
    t = time.time()
    eng.random_walk(ep, 0)
    t1 = time.time()
    ns = eng.build_samples(ep, 0)
    t2 = time.time()
    print(f"P={P} rank 0: walk {1e3*(t1-t):.1f} ms, build {1e3*(t2-t1):.1f} ms (host wall), pool {ns}", flush=True)
