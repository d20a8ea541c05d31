"""Benchmark: positive edge samples/s of the SGNS training path (BASELINE.json
metric) on B200, one process per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3] [--impl reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...

A step is one epoch of the whole hot path through the C ABI (ne_train_epoch):
walk engine -> window augmentation -> Feistel order + 2D bucketing -> SGNS
with K alias negatives, and at N > 1 the NCCL ring of vertex sub-parts.
`value` = positive samples trained by all ranks / max-over-ranks device time
(CUDA events on the library's compute stream), inputs resident in HBM.
`e2e` = the same metric with the CSR copied from pinned host memory every step
(ne_load_graph) and the step's loss read back (D2H).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "positive edge samples/sec at d=128, K=5 (1/2/4/8 B200); HBM GB/s vs peak"
UNIT = "positive samples/s"
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json
def sgns_kernel_name(d: int, K: int, bf16: bool) -> str:
    """The SGNS instantiation launch_sgns selects for (d, K, storage) -- the
    selection in sgns_kernel.cuh (launch_sgns_rows / launch_sgns_k)."""
    q = d // 4
    red = "bf16x4 red" if bf16 else "red.v4.f32"
    kt = 5 if K == 5 else 0
    if 16 < q <= 24 and K == 5:
        g, r, shape = 8, 3, "256x1"
    elif q <= 32:
        g, r, shape = 16, (1 if q <= 16 else 2), "256x2"
    else:
        g, r = 32, (q + 31) // 32
        shape = "256x2" if r == 2 else "64x1"
    return (f"ne::sgns_kernel<{g},{r},{kt},{shape},ADD,BF={int(bf16)}> ({g} lanes/sample, "
            f"{32 // g} samples/warp, {red} write-back)")


def alg_bytes_per_sample(d: int, K: int, esz: int = 4) -> int:
    """pair (8 B) + K alias entries (8 B) + read and write of the
    vertex row, the positive context row and K negative rows (2 esz d (2 + K);
    esz = 4 for fp32 rows: 7216 B at d = 128, K = 5; 2 for bf16 rows: 3632 B)."""
    return 8 + 8 * K + 2 * esz * d * (2 + K)


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def workload_desc(name):
    import synth
    w = synth.CONFIGS[name]
    gen = "R-MAT (Graph500 a,b,c=.57,.19,.19)" if w.kind == "rmat" else "uniform G(n,m)"
    return w, (f"{w.name} {gen} {w.n:,} nodes / {w.m:,} undirected edges "
               f"(nnz {2 * w.m:,}), " + (f"LINE edge pool, d={w.dim}, K={w.negatives}" if w.walk_len == 0 else
               f"{'DeepWalk' if (w.p, w.q) == (1.0, 1.0) else f'node2vec p={w.p} q={w.q}'} "
               f"k={w.walk_len} l={w.window} w=1, d={w.dim}, K={w.negatives}"))


def host_info() -> dict:
    """Host cores (nproc: the CPUs this process may run on) and CPU model."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"nproc": len(os.sched_getaffinity(0)), "cpu_model": model}


def oracle_hogwild(off, tgt, w, episodes: int, episode_ids, threads: int) -> dict:
    """The oracle's Hogwild timing mode (oracle/batch.c) on episodes
    `episode_ids` of an `episodes`-way split of epoch 0 of the workload, on
    full-size host matrices: pool built by one thread, SGNS by `threads`
    unsynchronised threads."""
    import oracle
    n = len(off) - 1
    cfg = oracle.Config(dim=w.dim, negatives=w.negatives, walk_len=w.walk_len, window=w.window,
                        walks_per_node=1, episodes=episodes, subparts=4, parts=1, seed=42, p=w.p, q=w.q)
    V = oracle.init_vertex(n, w.dim, 42)
    Cm = np.zeros_like(V)
    tables = oracle.build_alias_tables(cfg, off)
    tot = {"samples": 0, "sec_build": 0.0, "sec_train": 0.0, "per_step_s": []}
    for e in episode_ids:
        r = oracle.train_episode_hogwild(cfg, off, tgt, tables, V, Cm, 0, e, 0.025, threads)
        tot["samples"] += r["samples"]
        tot["sec_build"] += r["sec_build"]
        tot["sec_train"] += r["sec_train"]
        tot["per_step_s"].append(r["sec_build"] + r["sec_train"])
    return tot


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands (its Hogwild timing mode,
    one thread per host core), rank 0 only; each step is one episode of a
    --ref-episodes split of the workload's epoch 0."""
    if rank != 0:
        return
    import synth
    w, desc = workload_desc(args.workload)
    off, tgt = synth.workload_graph(args.workload)
    if not isinstance(off, np.ndarray):
        off, tgt = off.cpu().numpy().view(np.uint64), tgt.cpu().numpy().view(np.uint32)
    hi = host_info()
    T = hi["nproc"]
    E = args.ref_episodes
    oracle_hogwild(off, tgt, w, E, range(args.warmup), T)
    r = oracle_hogwild(off, tgt, w, E, range(args.warmup, args.warmup + args.steps), T)
    dt = r["sec_build"] + r["sec_train"]
    value = r["samples"] / dt
    sample = (f"episodes {args.warmup}..{args.warmup + args.steps - 1} of a {E}-episode split of epoch 0 "
              f"(~{(len(off) - 1) // E:,} walkers each, {r['samples']:,} positive samples timed), full-size "
              f"matrices; pool built by 1 thread ({r['sec_build']:.1f} s), SGNS by {T} Hogwild threads "
              f"({r['sec_train']:.1f} s)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
            "dtype": "f64 arithmetic, f32 storage", "data": "synthetic",
            "config": {"workload": desc, "impl": "oracle/ (plain C), Hogwild timing mode (oracle/batch.c)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": T, "threads": T, "kind": "oracle",
                             "sample": sample, **hi},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(args, off, tgt, w):
    """The oracle timed on this host on a bounded sample of the same workload:
    its Hogwild timing mode with one thread per host core over >= 10 M samples
    (one episode of a --cpu-episodes split), and beside it the deterministic
    single-thread path (the parity reference) on a smaller episode."""
    import oracle
    hi = host_info()
    T = hi["nproc"]
    n = len(off) - 1
    E = args.cpu_episodes
    r = oracle_hogwild(off, tgt, w, E, [0], T)
    dt = r["sec_build"] + r["sec_train"]
    # deterministic single thread (the parity reference), one episode of a 384-way split
    cfg = oracle.Config(dim=w.dim, negatives=w.negatives, walk_len=w.walk_len, window=w.window,
                        walks_per_node=1, episodes=384, subparts=4, parts=1, seed=42, p=w.p, q=w.q)
    V = oracle.init_vertex(n, w.dim, 42)
    Cm = np.zeros_like(V)
    tables = oracle.build_alias_tables(cfg, off)
    t0 = time.perf_counter()
    ns1, _ = oracle.train_epoch(cfg, off, tgt, V, Cm, 0, 0.025, 0, 1, tables=tables)
    dt1 = time.perf_counter() - t0
    return {"value": r["samples"] / dt, "unit": UNIT, "cores": T, "threads": T, "kind": "oracle", **hi,
            "sample": (f"episode 0 of a {E}-episode split of epoch 0 (~{n // E:,} walkers, {r['samples']:,} "
                       f"positive samples) on the full-size graph and matrices: pool built by 1 thread "
                       f"({r['sec_build']:.1f} s), SGNS by {T} Hogwild threads ({r['sec_train']:.1f} s)"),
            "sgns_only_value": r["samples"] / r["sec_train"],
            "deterministic_single_thread": {"value": ns1 / dt1, "unit": UNIT, "cores": 1,
                                            "sample": f"episode 0 of 384 ({ns1:,} samples: walk + pool + "
                                                      f"SGNS), {dt1:.1f} s"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-episodes", type=int, default=48, help="cpu_baseline: one episode of this split "
                    "(48: ~10.9 M samples on C3)")
    ap.add_argument("--ref-episodes", type=int, default=192, help="--impl reference: one episode per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--episodes", type=int, default=0, help="episodes per epoch (0 = workload default)")
    ap.add_argument("--subparts", type=int, default=4, help="vertex sub-parts per GPU (the paper's k, P:152)")
    ap.add_argument("--staging", default="device", choices=["device", "host"],
                    help="vertex matrix in HBM (device) or in pinned host memory streamed through device slots "
                         "(host: NEXT-2, the paper's pipeline stages 2 and 5, P:142)")
    ap.add_argument("--rule", default="sequential", choices=["sequential", "accumulated", "batch"],
                    help="update rule: Alg. 1 sequential (the headline), accumulated (word2vec), or batch "
                         "(NEXT-4 shared negatives: 128-sample batches share 32 negatives, tcgen05 tf32)")
    ap.add_argument("--transport", default="auto", choices=["auto", "nccl", "ipc"],
                    help="ring transport at N > 1: NCCL send/recv kernels, or copy-engine pushes over CUDA IPC; "
                         "auto = ipc (measured faster at every N and workload, profiles/r02_bench_*_ipc_*), "
                         "nccl with --staging host (the staged ring runs over NCCL)")
    ap.add_argument("--groups", type=int, default=1, help="NEXT-3 two-level ring: groups of N/groups ranks")
    ap.add_argument("--storage", default="f32", choices=["f32", "bf16"],
                    help="row storage: f32 (the paper's, the headline) or bf16 (NEXT-4 option, reading D16)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import synth
    from paper_2005_13789_b200 import ne
    from paper_2005_13789_b200.engine import Engine

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w, desc = workload_desc(args.workload)
    off, tgt = synth.workload_graph(args.workload, device=f"cuda:{local}")
    n = len(off) - 1
    episodes = args.episodes or w.episodes
    nccl_id = None
    if world > 1:
        obj = [ne.ne_get_nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    # the library computes on a dedicated torch stream; the timing events are
    # recorded on that same stream (ne_join first folds the ring's trailing
    # transfers, left on the library's comm stream, into it)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    if args.transport == "auto":
        args.transport = "nccl" if args.staging == "host" else "ipc"
    rule = {"sequential": ne.NE_UPDATE_SEQUENTIAL, "accumulated": ne.NE_UPDATE_ACCUMULATED,
            "batch": ne.NE_UPDATE_SHARED_BATCH}[args.rule]
    negatives = 32 if args.rule == "batch" else w.negatives
    eng = Engine(dim=w.dim, negatives=negatives, walk_len=w.walk_len, window=w.window,
                 walks_per_node=1, episodes=episodes, subparts=args.subparts, deterministic=False, seed=42,
                 update_rule=rule, staging=ne.NE_STAGE_HOST if args.staging == "host" else ne.NE_STAGE_DEVICE,
                 transport=ne.NE_TRANSPORT_IPC if args.transport == "ipc" else ne.NE_TRANSPORT_NCCL, groups=args.groups,
                 p=w.p, q=w.q, storage=ne.NE_STORE_BF16 if args.storage == "bf16" else ne.NE_STORE_F32,
                 device=local, rank=rank, world=world, nccl_id=nccl_id, torch_allocator=True,
                 stream=stream.cuda_stream)
    def all_gather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    eng.load_graph(off, tgt, all_gather=all_gather if world > 1 else None)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for s in range(args.warmup):
        eng.train_epoch(s, 0.025)
    barrier()
    stats = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        ev0.record(stream)
        for s in range(args.steps):
            stats.append(eng.train_epoch(args.warmup + s, 0.025))
        eng.join()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    samples = sum(st["samples"] for st in stats)
    ms_train = sum(st["ms_train"] for st in stats)
    launches = sum(st["kernel_launches"] for st in stats)
    train_launches = sum(st["train_launches"] for st in stats)
    t = torch.tensor([ms, samples, ms_train, launches, sum(st["ms_walk"] for st in stats),
                      sum(st["ms_build"] for st in stats), sum(st["ms_comm_wait"] for st in stats),
                      train_launches, sum(st["ms_pool_wait"] for st in stats)], dtype=torch.float64, device="cuda")
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    else:
        tmax = tsum = t
    ms_max = float(tmax[0])
    samples_all = float(tsum[1])
    value = samples_all / (ms_max / 1e3)

    # roofline of the dominant kernel (SGNS), this rank's launches
    esz = 2 if args.storage == "bf16" else 4
    B = alg_bytes_per_sample(w.dim, w.negatives, esz)
    if args.rule == "batch":  # per sample: pair, its vertex + positive rows (read + write), 32/128 of a shared
        B = 8 + 8 * 32 / 128 + 2 * esz * w.dim * (2 + 32 / 128)  # negative row and of its alias entry
    achieved = samples * B / (ms_train / 1e3) / 1e9 if ms_train > 0 else 0.0
    peak, peak_src = hbm_peak()
    traffic = dram_achieved = None
    prof = os.path.join(ROOT, "profiles", "sgns_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            tr = json.load(f).get(args.workload)
        key = ("batch_dram_bytes_per_sample" if args.rule == "batch" else
               "dram_bytes_per_sample" if esz == 4 else "bf16_dram_bytes_per_sample")
        per_sample = (tr or {}).get(key)
        if per_sample and train_launches:
            # captured DRAM bytes per sample x this run's samples per SGNS launch (this rank)
            traffic = per_sample * samples / train_launches
            dram_achieved = per_sample * samples / (ms_train / 1e3) / 1e9

    # end-to-end through the public API with host buffers (pinned): every step
    # loads the CSR from the host (H2D), trains one epoch, reads the loss and
    # copies this rank's trained vertex and context rows back to the host (D2H)
    if isinstance(off, np.ndarray):
        off_h = torch.from_numpy(off.view(np.int64)).pin_memory()
        tgt_h = torch.from_numpy(tgt.view(np.int32)).pin_memory()
    else:  # GPU-generated workload: stage it in pinned host memory for the e2e leg
        off_h, tgt_h = off.cpu().pin_memory(), tgt.cpu().pin_memory()
        del off, tgt
        torch.cuda.empty_cache()
        off, tgt = off_h.numpy().view(np.uint64), tgt_h.numpy().view(np.uint32)
    h2d = off_h.numel() * 8 + tgt_h.numel() * 4
    a, b = eng.part
    emb_h = [torch.empty((b - a, w.dim), dtype=torch.float32).pin_memory() for _ in range(2)]
    # fp32 rows in HBM: the vertex rows stream out during the epoch (ne_export_vertex_on_train:
    # one GPU, after the last episode's block; ring, on arrival home); otherwise read after it
    export_v = esz == 4 and args.staging == "device"
    if export_v:
        ne.ne_export_vertex_on_train(eng.ctx, emb_h[0])
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_samples = 0
    e0.record(stream)
    e_ph = {"load": 0.0, "train": 0.0, "get": 0.0}  # host-side split (each call returns synchronised)
    for s in range(args.e2e_steps):
        t0 = time.perf_counter()
        ne.ne_load_graph(eng.ctx, off_h, tgt_h)
        t1 = time.perf_counter()
        st = eng.train_epoch(s, 0.025)  # loss_sum / samples read back (D2H) by the call
        t2 = time.perf_counter()
        for which in ((ne.NE_CONTEXT,) if export_v else (ne.NE_VERTEX, ne.NE_CONTEXT)):
            ne.ne_get_embeddings(eng.ctx, which, a, b, emb_h[which])
        t3 = time.perf_counter()
        e_ph["load"] += (t1 - t0) * 1e3
        e_ph["train"] += (t2 - t1) * 1e3
        e_ph["get"] += (t3 - t2) * 1e3
        e_samples += st["samples"]
    e1.record(stream)
    barrier()
    d2h = 2 * (b - a) * w.dim * 4
    e_ms = torch.tensor([e0.elapsed_time(e1), e_samples], dtype=torch.float64, device="cuda")
    if world > 1:
        em = e_ms.clone()
        dist.all_reduce(em, op=dist.ReduceOp.MAX)
        es = e_ms.clone()
        dist.all_reduce(es, op=dist.ReduceOp.SUM)
        e_value = float(es[1]) / (float(em[0]) / 1e3)
    else:
        e_value = e_samples / (float(e_ms[0]) / 1e3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and w.m <= 200_000_000:
        cpu = cpu_baseline(args, off, tgt, w)
    eng.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": ("f32 rows, tf32 tensor-core products (NEXT-4 shared-negative batches; not the headline)"
                      if args.rule == "batch" else
                      "f32" if esz == 4 else "bf16 rows, f32 arithmetic (NEXT-4 option; not the headline)"),
            "data": "synthetic",
            "config": {"workload": desc, "step": "one epoch: walk + augment + order/bucket + SGNS (+ ring)",
                       "samples_per_step": samples_all / args.steps, "episodes": episodes, "subparts": args.subparts,
                       "update_rule": args.rule + (" (K'=32 negatives shared per 128-sample batch)"
                                                   if args.rule == "batch" else ""),
                       "staging": args.staging,
                       "mode": "hogwild",
                       "parallelism": f"2D ring x{world}" + (f" in {args.groups} groups" if args.groups > 1 else "")
                                      + (" (copy-engine IPC ring)" if args.transport == "ipc" and world > 1 else ""),
                       "l2": "inputs larger than L2 (embeddings %.2f GB vs 126 MB L2)" % (2 * n * w.dim * esz / 1e9),
                       "graph_generator": "numpy Philox (host)" if w.m <= 200_000_000 else "torch CUDA generator"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         # HBM-honest companion of frac: captured DRAM bytes per sample (ncu, committed
                         # profile) x this run's samples / SGNS time -- frac counts L2 hits as HBM bytes
                         "dram_achieved": dram_achieved,
                         "dram_frac": dram_achieved / peak if dram_achieved else None,
                         "kernel": ("ne::sgns_batch_kernel<128,32> (tcgen05.mma kind::tf32, TMEM accumulators)"
                                    if args.rule == "batch" else sgns_kernel_name(w.dim, w.negatives, esz == 2)),
                         "bytes_per_sample": B, "launches": train_launches,
                         "avg_launch_ms": ms_train / max(train_launches, 1), "peak_source": peak_src},
            "phases_ms_per_step": {"walk": float(tsum[4]) / world / args.steps,
                                   "build": float(tsum[5]) / world / args.steps,
                                   "train": float(tsum[2]) / world / args.steps,
                                   "comm_wait": float(tsum[6]) / world / args.steps,
                                   # walk + build time the compute stream waited for (the rest ran
                                   # on the build stream behind training)
                                   "pool_wait_exposed": float(tsum[8]) / world / args.steps},
            "cpu_baseline": cpu,
            "e2e": {"value": e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    # trained vertex + context rows of rank 0, CSR validation flags + offsets ends (32 B),
                    # block offsets, pool size and loss per episode
                    "d2h_bytes_per_step": d2h + 32 + episodes * (8 * (args.subparts * world + 1) + 16),
                    "step": "ne_load_graph (pinned host CSR) + ne_train_epoch + ne_get_embeddings of both "
                            "matrices (this rank's rows, to pinned host memory)"
                            + ("; the vertex rows stream out during the epoch as their sub-parts become "
                               "final (ne_export_vertex_on_train)" if export_v else ""),
                    "phases_ms_per_step": {k: v / max(1, args.e2e_steps) for k, v in e_ph.items()}},
            "clocks": clk.summary(),
            "gpu_launches": int(tsum[3]),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
