"""Convenience wrapper over the ne.h binding (argument marshalling only)."""
from __future__ import annotations

import numpy as np

from . import ne


class Engine:
    """One training context (one GPU / rank).  All compute runs in libne_b200.so."""

    def __init__(self, dim=128, negatives=5, walk_len=40, window=5, walks_per_node=1, episodes=1,
                 subparts=4, deterministic=False, seed=42, device=0, rank=0, world=1,
                 nccl_id=None, torch_allocator=False, stream=None, conflict_permille=0,
                 writeback=ne.NE_WB_ATOMIC_DELTA, p=1.0, q=1.0, update_rule=ne.NE_UPDATE_SEQUENTIAL,
                 staging=ne.NE_STAGE_DEVICE, storage=ne.NE_STORE_F32, transport=ne.NE_TRANSPORT_NCCL,
                 groups=1, stage_window=0):
        self.cfg = ne.ne_config(dim, negatives, walk_len, window, walks_per_node, episodes, subparts,
                                int(bool(deterministic)), conflict_permille, writeback, p, q, update_rule,
                                staging, storage, transport, seed, stage_window, groups)
        self._alloc = ne.torch_allocator() if torch_allocator else (None, None)
        self.ctx = ne.ne_create(self.cfg, device, *self._alloc)
        self.rank, self.world = rank, world
        if stream is not None:
            ne.ne_set_stream(self.ctx, stream)
        if world > 1 or rank != 0:
            ne.ne_init_dist(self.ctx, rank, world, nccl_id)
        self.n = 0

    # ---- graph
    def load_graph(self, offsets, targets, all_gather=None):
        """all_gather(bytes) -> [bytes per rank] (e.g. torch.distributed
        all_gather_object): needed by the IPC transport to connect the ring."""
        ne.ne_load_graph(self.ctx, offsets, targets)
        self.n = len(offsets) - 1
        self.bounds = ne.ne_partition_bounds(self.n, self.world).astype(np.int64)
        if self.cfg.transport == ne.NE_TRANSPORT_IPC and self.world > 1:
            if all_gather is None:
                raise ValueError("the IPC transport needs all_gather to exchange the ring handles")
            ne.ne_ipc_connect(self.ctx, all_gather(ne.ne_ipc_export(self.ctx)))

    @property
    def part(self) -> tuple[int, int]:
        return int(self.bounds[self.rank]), int(self.bounds[self.rank + 1])

    # ---- walk engine / pool
    def random_walk(self, epoch: int, episode: int, export: bool = False):
        if not export:
            return ne.ne_random_walk(self.ctx, epoch, episode, None)
        E = self.cfg.episodes
        U = self.n * self.cfg.walks_per_node
        units = (episode + 1) * U // E - episode * U // E
        out = np.zeros((units, self.cfg.walk_len + 1), np.uint32)
        ne.ne_random_walk(self.ctx, epoch, episode, out)
        return out

    def build_samples(self, epoch: int, episode: int) -> int:
        return ne.ne_build_samples(self.ctx, epoch, episode)

    def export_samples(self, vsub: int) -> np.ndarray:
        cnt = ne.ne_export_samples(self.ctx, vsub, None)
        out = np.zeros((max(cnt, 1), 2), np.uint32)
        ne.ne_export_samples(self.ctx, vsub, out)
        return out[:cnt]

    def export_negatives(self, epoch: int, episode: int, vsub: int, pos_begin: int, count: int) -> np.ndarray:
        out = np.zeros((max(count, 1), self.cfg.negatives), np.uint32)
        ne.ne_export_negatives(self.ctx, epoch, episode, vsub, pos_begin, count, out)
        return out[:count]

    def capture_block(self, epoch: int, episode: int, vsub: int, lr: float) -> np.ndarray:
        cnt = ne.ne_capture_block(self.ctx, epoch, episode, vsub, lr, None)
        out = np.zeros((max(cnt, 1), 2 + self.cfg.negatives), np.uint32)
        ne.ne_capture_block(self.ctx, epoch, episode, vsub, lr, out)
        return out[:cnt]

    # ---- training
    def train_samples(self, epoch: int, episode: int, lr: float) -> dict:
        return ne.ne_train_samples(self.ctx, epoch, episode, lr).as_dict()

    def train_epoch(self, epoch: int, lr: float, reuse: bool = False) -> dict:
        return ne.ne_train_epoch(self.ctx, epoch, lr, ne.NE_REUSE_SAMPLES if reuse else 0).as_dict()

    def join(self) -> None:
        ne.ne_join(self.ctx)

    # ---- embeddings
    def embeddings(self, which: int = ne.NE_VERTEX, rows: tuple[int, int] | None = None) -> np.ndarray:
        a, b = rows if rows is not None else self.part
        out = np.zeros((b - a, self.cfg.dim), np.float32)
        if b > a:
            ne.ne_get_embeddings(self.ctx, which, a, b, out)
        return out

    def export_vertex_on_train(self, out) -> None:
        """Every later train_epoch streams this rank's vertex rows into `out`
        (float32 [part rows][d], pinned for the overlap) while it trains; None
        turns it off.  The engine keeps a reference to `out`."""
        ne.ne_export_vertex_on_train(self.ctx, out)
        self._export = out

    def set_embeddings(self, which: int, row_begin: int, data: np.ndarray) -> None:
        data = np.ascontiguousarray(data, np.float32)
        ne.ne_set_embeddings(self.ctx, which, row_begin, row_begin + data.shape[0], data)

    def close(self):
        if self.ctx:
            ne.ne_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
