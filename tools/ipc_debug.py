"""torchrun worker: the smallest IPC-ring run with progress prints (debugging)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from paper_2005_13789_b200 import ne  # noqa: E402
from paper_2005_13789_b200.engine import Engine  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
torch.cuda.set_device(dev)
dist.init_process_group("gloo")


def log(*a):
    print(f"[rank {rank} {time.time() % 1000:.2f}]", *a, flush=True)


def all_gather(b):
    out = [None] * world
    dist.all_gather_object(out, b)
    return out


off, tgt = synth.rmat_graph(500, 3000, 11)
groups = int(sys.argv[1]) if len(sys.argv) > 1 else 1
eng = Engine(dim=32, walk_len=6, window=2, episodes=1, subparts=2, deterministic=True, device=dev, rank=rank,
             world=world, nccl_id=None, transport=ne.NE_TRANSPORT_IPC, groups=groups)
log("created")
eng.load_graph(off, tgt, all_gather=all_gather)
log("loaded + connected")
for ep in range(2):
    st = eng.train_epoch(ep, 0.025)
    log("epoch", ep, st["samples"], st["loss_sum"])
V = eng.embeddings(0)
log("embeddings", V.shape)
dist.barrier()
eng.close()
log("closed")
