#!/usr/bin/env python
"""Benchmark: PGA node-updates/s (n * B * l * iters / s) and best cut — BASELINE.json.

Default workload (N=1): BASELINE.json configs[1] — Barabasi-Albert n=10k m=4
(networkx, seed 0), B=1024 initialisations per GPU, full pDECO: 2 alternations x
(3 unlifted batches + 3 lifted batches, l=2), T=500 each, alpha=0.05, mu=0.9, IDI,
early exit off (work counted with early_exit=false on both sides).
One step = one full pDECO solve = 9.216e10 node-updates per GPU.

N>1 (torchrun, one process per GPU): members are sharded (rank r owns global
members [r*B, (r+1)*B)), so the job is the reference's solve with batch 1024*N;
per batch one NCCL allreduce(max) of the packed (cut, member) key and one of the
winner bits.  Weak scaling.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--config c2|c1|c4|c5] [--precision fp32|fp64]
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PGA node-updates/s (n*B*iters/s) and best cut value at 1/2/4/8 B200"
UNIT = "node-updates/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ workloads
def ba_graph(n, m, seed):
    import networkx as nx

    from paper_2509_18612_b200 import liftcut as lc

    G = nx.barabasi_albert_graph(n, m, seed=seed)
    e = np.array(G.edges(), dtype=np.int64)
    return _graph(n, e)


def er_sparse(n, avg_deg, seed):
    """G(n, p) with p = avg_deg/(n-1), geometric skipping (numpy; networkx
    fast_gnp_random_graph's method) — for config 4."""
    from paper_2509_18612_b200 import liftcut as lc

    rng = np.random.default_rng(seed)
    p = avg_deg / (n - 1)
    total = n * (n - 1) // 2
    k = int(total * p * 1.2) + 1000
    gaps = rng.geometric(p, size=k).astype(np.int64)
    idx = np.cumsum(gaps) - 1
    idx = idx[idx < total]
    # pair index -> (u, v), u < v, row-major
    u = (n - 2 - np.floor(np.sqrt(-8.0 * idx + 4.0 * n * (n - 1) - 7) / 2.0 - 0.5)).astype(np.int64)
    v = idx + u + 1 - n * (n - 1) // 2 + (n - u) * ((n - u) - 1) // 2
    return _graph(n, np.stack([u, v], 1))


def _graph(n, edges):
    """Graph(n, edges): on the device (lcb_graph_from_edges) when a GPU is present, else
    the host constructor; both give the same CSR (tests/test_gpu_ingest.py)."""
    from paper_2509_18612_b200 import liftcut as lc
    import torch

    if torch.cuda.is_available():
        return lc.Graph.from_edges_device(n, edges)
    return lc.Graph(n, edges)


def workload(name, nranks, precision):
    from paper_2509_18612_b200 import liftcut as lc

    if name == "c1":
        g = lc.generate_er(800, 0.015, 0)
        cfg = lc.SolverConfig(algorithm=lc.Algorithm.pQUCO, batch_size=64,
                              ascent=lc.AscentParams(0.05, 500, 0.9, False), num_batches=1)
        desc = "ER n=800 p=0.015 seed0 (ref generator), pQUCO B=64, T=500, 1 batch"
    elif name == "c3":
        g = lc.generate_er(20_000, 0.5, 0)
        cfg = lc.SolverConfig(algorithm=lc.Algorithm.pQUCO, batch_size=256,
                              ascent=lc.AscentParams(0.05, 500, 0.9, False), num_batches=1)
        desc = "dense ER n=20k p=0.5 (ref generator, ~1e8 edges), pQUCO B=256, T=500, tensor-core path"
    elif name == "c4":
        g = er_sparse(1_000_000, 10.0, 0)
        cfg = lc.SolverConfig(algorithm=lc.Algorithm.pQUCO, batch_size=512 // nranks if nranks > 1 else 512,
                              ascent=lc.AscentParams(0.05, 500, 0.9, False), num_batches=1)
        desc = "sparse ER n=1M avg deg 10, pQUCO B=512 global, T=500, 1 batch"
    elif name == "c5":
        g = ba_graph(100_000, 4, 0)
        cfg = lc.SolverConfig(algorithm=lc.Algorithm.pQUCO, batch_size=256,
                              ascent=lc.AscentParams(0.05, 500, 0.9, False), num_batches=1,
                              search=lc.auto_search_bounds())
        desc = ("BA n=100k m=4, pQUCO B=256 + evolutionary (alpha,T) search; at N GPUs N independent "
                "searches (seed k*N+rank), best cut reduced over ranks with NCCL")
    else:
        g = ba_graph(10_000, 4, 0)
        cfg = lc.SolverConfig(algorithm=lc.Algorithm.pDECO, batch_size=1024, lift_dim=2,
                              ascent=lc.AscentParams(0.05, 500, 0.9, False), num_batches=3,
                              deco_alternations=2)
        desc = ("Barabasi-Albert n=10k m=4 (networkx seed 0), B=1024/GPU, full pDECO "
                "(2 x [3 quco + 3 luco l=2 batches]), T=500, IDI, early exit off")
    return g, cfg, desc


def expected_updates(g, cfg) -> int:
    n, B, T = g.node_count(), cfg.batch_size, cfg.ascent.iterations
    if cfg.algorithm == 2:
        return n * T * cfg.num_batches * cfg.deco_alternations * (B + B * cfg.lift_dim)
    l = cfg.lift_dim if cfg.algorithm == 1 else 1
    return n * T * cfg.num_batches * B * l


# ------------------------------------------------------------------ helpers
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.rows, self.proc = [], None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7 for i in range(4)
                          if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def measured_tensor_peak():
    """Dense bf16 peak from MEASURED_PEAKS.json: the sustained figure (the dense
    kernel runs back to back for the whole step)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("bf16_tflops_sustained", d.get("bf16_tflops", 1590.0)), "measured (sustained)"
    return 1590.0, "fallback"


def ncu_traffic(config, precision, kernel):
    """dram__bytes_read + dram__bytes_write per launch of `kernel` from the committed
    ncu capture of this workload (profiles/ncu_summary.json), if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    e = d.get(f"{config}_{precision}_{kernel}")
    return e.get("dram_bytes_per_launch") if e else None


def cpu_reference_step(g, cfg, nranks, t_sample, repeats=1):
    """The reference's own CPU solve (oracle/_ref, unmodified liftcut compiled from
    /root/reference) on the same graph and config, T reduced to t_sample (or the full
    solve repeated `repeats` times for tiny configs), all host threads.
    Returns (node-updates, seconds, best cut, threads)."""
    import oracle as O

    rg = O.RefGraph.from_csr(O.CSR(g.node_count(), g.offsets, g.adjacency))
    c = cfg.to_abi()
    cc = O.default_config()
    for f, _ in O.Config._fields_:
        setattr(cc, f, getattr(c, f))
    cc.batch_size = cfg.batch_size * nranks
    cc.iterations = t_sample
    cc.l_iterations = t_sample
    cc.has_search = 0
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    best = 0
    for rep in range(repeats):
        best = max(best, O.ref_solve(rg, cc, rep, workers=threads).cut_value)
    dt = time.perf_counter() - t0
    from copy import deepcopy

    cfg2 = deepcopy(cfg)
    cfg2.batch_size = cfg.batch_size * nranks
    cfg2.ascent.iterations = t_sample
    cfg2.search = None
    return expected_updates(g, cfg2) * repeats, dt, best, threads


def ref_sample(name):
    """(T, repeats) of one bounded CPU sample: ~10-15 s of reference work on the GPU box's
    16 host threads (measured samples: c1 400 solves 6.8 s, c2 T=50 9.6 s, c3 T=1 10.2 s,
    c4 T=4 8.8 s, c5 T=200 5.3 s); per-batch init / rounding stays the share it has at the
    full T."""
    return {"c1": (500, 600), "c2": (55, 1), "c3": (1, 1), "c4": (5, 1), "c5": (400, 1)}[name]


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libliftcut_ref.so")):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libliftcut_ref.so not built"}))
        return 0
    g, cfg, desc = workload(args.config, args.gpus, args.precision)
    T, reps = ref_sample(args.config)
    for _ in range(args.warmup):
        cpu_reference_step(g, cfg, args.gpus, 1)  # cache warm-up only
    ups, secs, best = 0, 0.0, 0
    threads = 1
    for _ in range(args.steps):
        u, dt, cut, threads = cpu_reference_step(g, cfg, args.gpus, T, reps)
        ups += u
        secs += dt
        best = max(best, cut)
    value = ups / secs
    sample = (f"reference pDECO/pQUCO solve with T={T} (of {cfg.ascent.iterations}), global batch "
              f"{cfg.batch_size * args.gpus}" + (f", {reps} solves per step" if reps > 1 else ""))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "best_cut": best,
        "config": {"workload": desc + f" [reference CPU sample: T={T}" + (f" x {reps} solves" if reps > 1 else "") + "]", "graph_nodes": g.node_count(),
                   "graph_edges": g.edge_count()},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


# ------------------------------------------------------------------ B200 arm
def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2509_18612_b200 import LCB_FP32, LCB_FP64
    from paper_2509_18612_b200 import liftcut as lc
    from paper_2509_18612_b200.dist import Comm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ["LIFTCUT_DEVICE"] = str(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = Comm.from_torch(local)
    prec = LCB_FP32 if args.precision == "fp32" else LCB_FP64
    g, cfg, desc = workload(args.config, world, args.precision)
    # batched search rounds measured slower on config 5 (B=256 already fills the GPU; see
    # profiles/round1_kernel_ab.md), so the bench keeps the sequential evolve() order
    # config 5 shards independent searches: rank r runs its own solve with seed
    # k*N + r and no member sharding; the best cut is reduced over ranks with NCCL at the end
    independent = args.config == "c5" and world > 1
    opts = lc.RunOptions(precision=prec, host_init=0, comm=None if independent else comm, batched_search=False)
    seed_of = (lambda k: k * world + rank) if independent else (lambda k: k)
    solve = {0: lc.pquco, 1: lc.pluco, 2: lc.pdeco}[int(cfg.algorithm)]
    g.handle(local)  # inputs resident in HBM before timing

    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        solve(g, cfg, seed=0, opts=opts)
    barrier()

    sampler = ClockSampler(local) if rank == 0 else None
    l0 = lc.counters()[0]
    dev_ms, step_ms, step_bytes, launches, ups, best = 0.0, 0.0, 0.0, 0, 0, 0
    kst = {"k_step": [0.0, 0.0, 0.0], "k_resident": [0.0, 0.0, 0.0], "k_dense_step": [0.0, 0.0, 0.0]}
    for k in range(args.steps):
        flush.fill_(k & 0xFF)  # L2 flush between timed steps (untimed)
        barrier()
        out = solve(g, cfg, seed=seed_of(k), opts=opts)
        dev_ms += out.solve_ms
        step_ms += out.step_ms
        step_bytes += out.step_bytes
        launches += out.step_launches
        for kname, vals in out.kernel_stats.items():
            for i in range(3):
                kst[kname][i] += vals[i]
        ups += out.node_updates
        best = max(best, out.best.cut_value)
        if lc.cut_value(g, out.best.assignment) != out.best.cut_value:
            raise RuntimeError("reported cut does not recompute")
    barrier()
    gpu_launches = lc.counters()[0] - l0
    clocks = sampler.stop() if sampler else None

    # e2e: the public API with HOST buffers (graph upload + assignment download inside)
    h0, d0 = lc.counters()[1:]
    barrier()
    t0 = time.perf_counter()
    for k in range(args.steps):
        gh = lc.Graph.from_csr(g.node_count(), g.offsets, g.adjacency)
        solve(gh, cfg, seed=seed_of(k), opts=opts)
        gh.release()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    h1, d1 = lc.counters()[1:]

    t = torch.tensor([dev_ms, e2e_s], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms, max_e2e = float(t[0]), float(t[1])
    if world > 1:  # best cut over ranks (identical on every rank unless the runs are independent)
        bt = torch.tensor([best], dtype=torch.int64, device=f"cuda:{local}")
        dist.all_reduce(bt, op=dist.ReduceOp.MAX)
        best = int(bt[0])
    total_ups = ups * world
    value = total_ups / (max_ms / 1e3)
    e2e_value = total_ups / max_e2e

    if rank == 0:
        peak, which = measured_peaks()
        # roofline of the dominant step kernel (largest share of step-kernel time)
        kname = max(kst, key=lambda k: kst[k][0])
        k_ms, k_launch, k_amount = kst[kname]
        shares = {k: v[0] / max(step_ms, 1e-9) for k, v in kst.items() if v[1]}
        if kname == "k_dense_step":
            tpeak, twhich = measured_tensor_peak()
            achieved = k_amount / (k_ms / 1e3) / 1e12
            roof = {"bound": "tensor", "achieved": achieved, "peak": tpeak, "unit": "TFLOP/s",
                    "frac": achieved / tpeak, "traffic": ncu_traffic(args.config, args.precision, kname),
                    "kernel": kname, "algorithmic_flops_per_launch": k_amount / max(k_launch, 1),
                    "ms_per_launch": k_ms / max(k_launch, 1), "step_time_share": shares, "peak_source": twhich,
                    "model": "2*n^2*W algorithmic flops per iteration (SURVEY 8d). Executed MMA work differs "
                             "per 32-node K step: bf16 hi/mid/lo planes before saturation, mid/lo skipped when "
                             "all zero, e4m3 MMAs on corner-valued steps (DESIGN.md K3)"}
        else:
            achieved = k_amount / (k_ms / 1e3) / 1e9
            roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": ncu_traffic(args.config, args.precision, kname),
                    "kernel": kname, "algorithmic_bytes_per_launch": k_amount / max(k_launch, 1),
                    "ms_per_launch": k_ms / max(k_launch, 1), "step_time_share": shares, "peak_source": which,
                    "model": "16 B/node-update fp32 (32 fp64) + CSR bytes per iteration (SURVEY 8d)"}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            T, reps = ref_sample(args.config)
            try:
                u, dt, _, thr = cpu_reference_step(g, cfg, 1, T, reps)
                cpu = {"value": u / dt, "unit": UNIT, "cores": thr, "kind": "reference",
                       "sample": f"unmodified reference solve (oracle/_ref) of the same graph/config with "
                                 f"T={T} instead of {cfg.ascent.iterations}"
                                 + (f", {reps} solves" if reps > 1 else "") + f", {thr} host threads, {dt:.1f} s"}
            except Exception as e:  # noqa: BLE001
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if prec == LCB_FP32 else "f64", "data": "synthetic",
            "best_cut": best,
            "config": {"workload": desc, "config_id": args.config, "graph_nodes": g.node_count(),
                       "graph_edges": g.edge_count(), "members_per_gpu": cfg.batch_size,
                       "global_batch": cfg.batch_size * world,
                       "node_updates_per_step": total_ups // args.steps,
                       "l2": "flushed between timed steps (512 MB write); each step is a full solve",
                       "parallelism": f"member-sharded dp{world}" if world > 1 else "single GPU",
                       "timing": "CUDA events on the solver stream, sum over steps, max over ranks"},
            "roofline": roof,
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": (h1 - h0) // args.steps,
                    "d2h_bytes_per_step": (d1 - d0) // args.steps},
            "gpu_launches": gpu_launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
