"""Quick perf probe: time walk/build/train of one epoch on a workload."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import synth
from paper_2005_13789_b200.engine import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
subparts = int(sys.argv[3]) if len(sys.argv) > 3 else 4
rule = int(sys.argv[4]) if len(sys.argv) > 4 else 0
storage = int(sys.argv[5]) if len(sys.argv) > 5 else 0  # 1 = bf16 rows (NEXT-4)
t = time.time()
off, tgt = synth.workload_graph(name, device="cuda")
print(f"{name}: graph n={len(off)-1} nnz={len(tgt)} gen {time.time()-t:.1f}s", flush=True)
import torch
if torch.cuda.is_available(): print(f"after gen: {torch.cuda.mem_get_info()[0]/1e9:.1f} GB free", flush=True)
w = synth.CONFIGS[name]
import torch
eng = Engine(dim=w.dim, deterministic=False, episodes=w.episodes, p=w.p, q=w.q, subparts=subparts, update_rule=rule,
             storage=storage, negatives=32 if rule == 2 else 5)  # rule 2: 32 shared negatives per batch of 128
t = time.time(); eng.load_graph(off, tgt); print(f"load {time.time()-t:.2f}s  mem {torch.cuda.mem_get_info()[0]/1e9:.1f} GB free", flush=True)
del off, tgt
torch.cuda.empty_cache()
for ep in range(epochs):
    t = time.time()
    st = eng.train_epoch(ep, 0.025)
    wall = time.time() - t
    B = 8 + 8 * 5 + (4 if storage else 8) * w.dim * 7
    if rule == 2:  # per sample: pair, vertex + positive rows read and written, 32/128 of a shared negative row
        B = 8 + 8 * 32 / 128 + 8 * w.dim * (2 + 32 / 128)
    print(f"k={subparts} rule={rule} epoch {ep}: wall {wall:.3f}s samples {st['samples']} walk {st['ms_walk']:.1f}ms build {st['ms_build']:.1f}ms "
          f"train {st['ms_train']:.1f}ms exposed-build {st['ms_pool_wait']:.1f}ms -> {st['samples']/st['ms_train']/1e3:.1f} M samples/s kernel, "
          f"{st['samples']*B/st['ms_train']/1e6:.0f} GB/s alg; loss/sample {st['loss_sum']/max(st['samples'],1)/6:.4f}", flush=True)
