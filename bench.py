#!/usr/bin/env python
"""Benchmark: PGA node-updates/s (n * B * l * iters / s) and best cut — BASELINE.json.

Headline (default, N=1): BASELINE.json config 4 — sparse ER n=1M, average degree 10
(networkx fast_gnp_random_graph(n, 10/(n-1), seed 0), m = 4,999,707), B=512
initialisations per GPU, pQUCO, T=500, alpha=0.05, mu=0.9, IDI, early exit off (BASELINE.md:
work counted with early_exit=false on both sides), fp32.  The largest single-GPU
configuration and the one BASELINE shards over 1/2/4/8 GPUs.  One step = one full
solve = 2.56e11 node-updates per GPU.

N>1 (one process per GPU; without WORLD_SIZE, `--gpus N` launches torch.distributed.run
itself): members are sharded (rank r owns global members [r*B, (r+1)*B)), so the job is
the reference's solve with batch 512*N; per batch one NCCL allreduce(max) of the packed
(cut, member) key and one of the winner bits.  Weak scaling.

At N=1 the same JSON line also carries `extra_configs`: configs 2, 3, 5 (fp32) and the
headline in fp64 (the bit-exact mode), each measured in this run with fewer steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--config c4|c1|c2|c3|c5] [--precision fp32|fp64] [--no-extras]

`--impl reference` times the reference's own CPU solver (oracle/_ref: the unmodified
/root/reference sources compiled in-tree) on the host cores, on a bounded T sample of the
same workload; its process never imports the B200 package (graphs from the same
generators through the reference's constructor / generate_er).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import random
import socket
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
DEFAULT_CONFIG = "c4"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ graphs (no product import)
def fast_gnp_edges(n, p, seed):
    """networkx.fast_gnp_random_graph(n, p, seed) (Batagelj-Brandes skipping), vectorised:
    the same Mersenne-Twister stream as random.Random(seed), the same math.log and the same
    truncation, so the edge set is identical (checked against networkx in
    tests/test_bench_cpu.py); the skip sum is the linear index of pair (v, w), w < v."""
    rng = random.Random(seed)
    st = rng.getstate()[1]
    rs = np.random.RandomState()
    rs.set_state(("MT19937", np.array(st[:624], dtype=np.uint32), st[624]))
    lp = math.log(1.0 - p)
    total = n * (n - 1) // 2
    out, L = [], -1
    chunk = int(total * p * 1.05) + 1024
    while True:
        r = rs.random_sample(chunk)
        lr = np.fromiter((math.log(x) for x in (1.0 - r)), dtype=np.float64, count=chunk)
        idx = L + np.cumsum(1 + np.floor(lr / lp).astype(np.int64))
        L = int(idx[-1])
        done = idx >= total
        if done.any():
            out.append(idx[: int(np.argmax(done))])
            break
        out.append(idx)
    idx = np.concatenate(out)
    v = np.floor((1.0 + np.sqrt(1.0 + 8.0 * idx.astype(np.float64))) / 2.0).astype(np.int64)
    v -= (v * (v - 1) // 2 > idx)
    v += ((v + 1) * v // 2 <= idx)
    return v, idx - v * (v - 1) // 2


def ba_edges(n, m, seed):
    import networkx as nx

    e = np.array(nx.barabasi_albert_graph(n, m, seed=seed).edges(), dtype=np.int64)
    return e[:, 0], e[:, 1]


# ------------------------------------------------------------------ workloads
# lcb_config fields (SolverConfig defaults: IDI beta 0.2, eta 0.8, init_scale 1e4)
BASE = dict(algorithm=0, lift_dim=2, batch_size=64, num_batches=1, alpha=0.05, iterations=500, momentum=0.9,
            early_exit=0, has_lifted_ascent=0, l_alpha=0.05, l_iterations=500, l_momentum=0.9, l_early_exit=0,
            init_method=1, beta=0.2, eta=0.8, init_scale=1e4, init_seed=0, resample_idi=1, scale_noise=1,
            time_budget_s=0.0, has_search=0, population_size=6, t_lower=3000, t_upper=10000, e_lower=-4.0,
            e_upper=-1.0, rounds=5, search_refresh=0, deco_alternations=2, deco_carry=0)

WORKLOADS = {
    "c1": dict(graph=("er_ref", 800, 0.015, 0), cfg=dict(batch_size=64),
               desc="ER n=800 p=0.015 seed 0 (reference generate_er), pQUCO B=64/GPU, T=500, 1 batch"),
    "c2": dict(graph=("ba", 10_000, 4, 0),
               cfg=dict(algorithm=2, batch_size=1024, lift_dim=2, num_batches=3, deco_alternations=2),
               desc="Barabasi-Albert n=10k m=4 (networkx seed 0), B=1024/GPU, full pDECO "
                    "(2 x [3 quco + 3 luco l=2 batches]), T=500, IDI, early exit off"),
    "c3": dict(graph=("er_ref", 20_000, 0.5, 0), cfg=dict(batch_size=256),
               desc="dense ER n=20k p=0.5 seed 0 (reference generate_er, ~1e8 edges), pQUCO B=256/GPU, T=500, "
                    "tensor-core path"),
    "c4": dict(graph=("gnp", 1_000_000, 10.0 / 999_999, 0), cfg=dict(batch_size=512),
               desc="sparse ER n=1M avg degree 10 (networkx fast_gnp_random_graph seed 0, m=4,999,707), "
                    "pQUCO B=512/GPU, T=500, IDI, early exit off, 1 batch"),
    "c5": dict(graph=("ba", 100_000, 4, 0), cfg=dict(batch_size=256, has_search=1),
               desc="BA n=100k m=4 (networkx seed 0), pQUCO B=256 + evolutionary (alpha, T) search "
                    "(auto bounds: T in [3000, 10000], pop 6, 5 rounds); one independent run per GPU per step "
                    "(seed = step*N + rank), best cut reduced over ranks"),
}


def solver_fields(name):
    d = dict(BASE)
    d.update(WORKLOADS[name]["cfg"])
    return d


def graph_edges(name):
    kind, *a = WORKLOADS[name]["graph"]
    if kind == "gnp":
        return a[0], fast_gnp_edges(*a)
    if kind == "ba":
        return a[0], ba_edges(*a)
    raise ValueError(kind)


def config_dict(name, world, precision):
    """The `config` object of the JSON line — identical for both arms."""
    f = solver_fields(name)
    n = WORKLOADS[name]["graph"][1]
    l = f["lift_dim"] if f["algorithm"] else 1
    return {"workload": WORKLOADS[name]["desc"], "config_id": name, "precision": precision,
            "graph_nodes": n, "members_per_gpu": f["batch_size"], "global_batch": f["batch_size"] * world,
            "lift_dim": l, "iterations": f["iterations"],
            "parallelism": f"member-sharded dp{world}" if world > 1 and name != "c5" else
            (f"independent runs x{world}" if world > 1 else "single GPU"),
            "l2": "flushed between timed steps (512 MB write); each step is a full solve"}


def expected_updates(f, n) -> int:
    B, T = f["batch_size"], f["iterations"]
    if f["algorithm"] == 2:
        return n * T * f["num_batches"] * f["deco_alternations"] * (B + B * f["lift_dim"])
    l = f["lift_dim"] if f["algorithm"] == 1 else 1
    return n * T * f["num_batches"] * B * l


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


def ncu_entry(config, precision, kernel):
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        return json.load(f).get(f"{config}_{precision}_{kernel}", {})


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


def ref_sample(name):
    """(T, repeats) of one bounded CPU step: a few seconds of reference ascent on the GPU
    box's host cores (c1: whole solves, c3: 1 iteration of the 1e8-edge graph)."""
    return {"c1": (500, 40), "c2": (20, 1), "c3": (1, 1), "c4": (2, 1), "c5": (200, 1)}[name]


def cpu_reference_step(rg, name, world, T, reps, threads):
    """The reference's own solve (oracle/_ref: unmodified liftcut) on the same graph and
    config, T reduced to the sample, all host threads, no search.  Returns (node-updates,
    StageTimes.ascent_s, solve seconds, best cut)."""
    import oracle as O

    f = solver_fields(name)
    f["batch_size"] *= world
    f["iterations"] = f["l_iterations"] = T
    f["has_search"] = 0
    cc = O.default_config(**f)
    ups, asc, sec, best = 0, 0.0, 0.0, 0
    for rep in range(reps):
        t0 = time.perf_counter()
        r = O.ref_solve(rg, cc, rep, workers=threads)
        sec += time.perf_counter() - t0
        asc += r.stage_times["ascent_s"]
        best = max(best, r.cut_value)
        ups += expected_updates(f, rg.n)
    return ups, asc, sec, best


def cpu_single_thread(rg):
    """the reference's ascend on ONE host thread (the member-parallel reference
    scales with threads up to B): a few members, T=2, timed around ref_ascend."""
    import numpy as np

    import oracle as O

    B, T = 32, 2
    x = np.random.default_rng(0).uniform(-1e-4, 1e-4, B * rg.n)
    t0 = time.perf_counter()
    O.ref_ascend(rg, x, 1, B, 0.05, T, 0.9, False, workers=1)
    dt = time.perf_counter() - t0
    return rg.n * B * T / dt, f"reference ascend, {B} members x T={T}, 1 thread ({dt:.1f} s)"


def reference_graph(name):
    import oracle as O

    kind, *a = WORKLOADS[name]["graph"]
    if kind == "er_ref":
        return O.RefGraph.er(*a)
    n, (u, v) = graph_edges(name)
    return O.RefGraph.from_edges(n, u, v)


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libliftcut_ref.so")):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libliftcut_ref.so not built"}))
        return 0
    assert "paper_2509_18612_b200" not in sys.modules
    world = args.gpus
    rg = reference_graph(args.config)
    T, reps = ref_sample(args.config)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference_step(rg, args.config, world, 1, 1, threads)  # page-in / cache warm-up only
    ups, asc, sec, best = 0, 0.0, 0.0, 0
    for _ in range(args.steps):
        u, a, s, b = cpu_reference_step(rg, args.config, world, T, reps, threads)
        ups, asc, sec, best = ups + u, asc + a, sec + s, max(best, b)
    assert "paper_2509_18612_b200" not in sys.modules
    value = ups / asc
    f = solver_fields(args.config)
    sample = (f"unmodified reference solve (oracle/_ref, compiled from /root/reference) with T={T} instead of "
              f"{f['iterations']}, global batch {f['batch_size'] * world}, no search"
              + (f", {reps} solves per step" if reps > 1 else "")
              + f", {threads} host threads; value = node-updates / StageTimes.ascent_s "
                f"({asc:.1f} s of {sec:.1f} s solve wall; solve-wall rate {ups / sec:.3e})")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * asc / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "best_cut_sample": best, "config": config_dict(args.config, world, args.precision),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


# ------------------------------------------------------------------ B200 arm
class Arm:
    def __init__(self, world, rank, local, comm):
        self.world, self.rank, self.local, self.comm = world, rank, local, comm

    def barrier(self):
        import torch
        import torch.distributed as dist

        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()

    def allreduce_max(self, vals, dtype):
        import torch
        import torch.distributed as dist

        t = torch.tensor(vals, dtype=getattr(torch, dtype), device=f"cuda:{self.local}")
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()


def product_config(lc, f):
    a = lc.AscentParams(f["alpha"], f["iterations"], f["momentum"], bool(f["early_exit"]))
    la = (lc.AscentParams(f["l_alpha"], f["l_iterations"], f["l_momentum"], bool(f["l_early_exit"]))
          if f["has_lifted_ascent"] else None)
    init = lc.InitConfig(lc.InitMethod(f["init_method"]), f["beta"], f["eta"], f["init_scale"], f["init_seed"],
                         bool(f["resample_idi"]), bool(f["scale_noise"]))
    search = (lc.SearchConfig(f["t_lower"], f["t_upper"], f["e_lower"], f["e_upper"], f["population_size"],
                              f["rounds"]) if f["has_search"] else None)
    return lc.SolverConfig(lc.Algorithm(f["algorithm"]), f["batch_size"], f["lift_dim"], a, la, init,
                           f["num_batches"], None, search, f["search_refresh"], f["deco_alternations"],
                           lc.DecoCarry(f["deco_carry"]))


def device_graph(lc, name, device):
    kind, *a = WORKLOADS[name]["graph"]
    if kind == "er_ref":
        return lc.generate_er_device(*a, device=device)
    n, (u, v) = graph_edges(name)
    return lc.Graph.from_edges_device(n, np.stack([u, v], 1), device)


KERNELS = ("k_step", "k_resident", "k_dense_step", "k_stream")


def measure(arm, name, precision, steps, warmup, flush, with_e2e, host_init=0):
    import torch  # noqa: F401

    from paper_2509_18612_b200 import LCB_FP32, LCB_FP64
    from paper_2509_18612_b200 import liftcut as lc

    prec = LCB_FP32 if precision == "fp32" else LCB_FP64
    f = solver_fields(name)
    cfg = product_config(lc, f)
    g = device_graph(lc, name, arm.local)
    independent = name == "c5"  # independent runs, one per rank per step
    opts = lc.RunOptions(precision=prec, host_init=host_init, comm=arm.comm, batched_search=False)
    if independent:
        # the library shards the step's runs over the ranks and reduces the best cut and
        # its assignment with one exchange (lcb_solve_runs; bench.cpp:97-136)
        def solve(g, cfg, seed, opts):
            r = lc.solve_runs(g, cfg, [seed * arm.world + q for q in range(arm.world)], per_component=False,
                              opts=opts)
            r.node_updates_total = r.node_updates
            return r
    else:
        solve = {0: lc.pquco, 1: lc.pluco, 2: lc.pdeco}[f["algorithm"]]
    seed_of = lambda k: k  # noqa: E731
    g.handle(arm.local)  # inputs resident in HBM before timing
    if independent:  # warm-up without the search (one search solve is ~10 s)
        wcfg = product_config(lc, {**f, "has_search": 0, "iterations": 50})
        for _ in range(warmup):
            solve(g, wcfg, seed=1000, opts=opts)
    else:
        for _ in range(warmup):
            solve(g, cfg, seed=0, opts=opts)
    arm.barrier()
    l0 = lc.counters()[0]
    dev_ms, step_ms, ups, best = 0.0, 0.0, 0, 0
    kst = {k: [0.0, 0.0, 0.0] for k in KERNELS}
    for k in range(steps):
        flush.fill_(k & 0xFF)  # L2 flush between timed steps (untimed)
        arm.barrier()
        out = solve(g, cfg, seed=seed_of(k), opts=opts)
        dev_ms += out.solve_ms
        step_ms += out.step_ms
        for kname, vals in out.kernel_stats.items():
            for i in range(3):
                kst[kname][i] += vals[i]
        ups += out.node_updates
        best = max(best, out.best.cut_value)
        if lc.cut_value(g, out.best.assignment) != out.best.cut_value:
            raise RuntimeError("reported cut does not recompute")
    arm.barrier()
    launches = lc.counters()[0] - l0

    e2e_s, h2d, d2h = None, 0, 0
    if with_e2e:  # the public API with HOST buffers (graph upload + assignment download inside)
        h0, d0 = lc.counters()[1:]
        arm.barrier()
        t0 = time.perf_counter()
        for k in range(steps):
            gh = lc.Graph.from_csr(g.node_count(), g.offsets, g.adjacency)
            solve(gh, cfg, seed=seed_of(k), opts=opts)
            gh.release()
        arm.barrier()
        e2e_s = time.perf_counter() - t0
        h1, d1 = lc.counters()[1:]
        h2d, d2h = (h1 - h0) // steps, (d1 - d0) // steps

    mx = arm.allreduce_max([dev_ms, e2e_s or 0.0], "float64")
    best = int(arm.allreduce_max([best], "int64")[0]) if arm.world > 1 else best
    total_ups = ups * arm.world
    res = {"value": total_ups / (mx[0] / 1e3), "ms_per_step": mx[0] / steps, "best_cut": best,
           "node_updates_per_step": total_ups // steps, "gpu_launches": launches,
           "graph_nodes": g.node_count(), "graph_edges": g.edge_count(), "dtype": "f32" if prec == LCB_FP32 else "f64"}
    if e2e_s is not None:
        res["e2e"] = {"value": total_ups / mx[1], "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
    res["roofline"] = roofline(kst, step_ms, name, precision)
    g.release()
    return res


def roofline(kst, step_ms, name, precision):
    kname = max(kst, key=lambda k: kst[k][0])
    k_ms, k_launch, k_amount = kst[kname]
    shares = {k: v[0] / max(step_ms, 1e-9) for k, v in kst.items() if v[1]}
    if kname == "k_dense_step":
        tpeak, twhich = measured_tensor_peak()
        achieved = k_amount / (k_ms / 1e3) / 1e12
        return {"bound": "tensor", "achieved": achieved, "peak": tpeak, "unit": "TFLOP/s", "frac": achieved / tpeak,
                "traffic": ncu_traffic(name, precision, kname), "kernel": kname,
                "algorithmic_flops_per_launch": k_amount / max(k_launch, 1),
                "ms_per_launch": k_ms / max(k_launch, 1), "step_time_share": shares, "peak_source": twhich,
                "tensor_pipe_active_pct": ncu_entry(name, precision, kname).get("tensor_pipe_active_pct"),
                "model": "2*n^2*W algorithmic flops per iteration (SURVEY 8d). Executed MMA work differs per "
                         "32-node K step: bf16 hi/mid/lo planes before saturation, mid/lo skipped when all zero, "
                         "e4m3 MMAs on corner-valued steps (DESIGN.md K3)"}
    peak, which = measured_peaks()
    achieved = k_amount / (k_ms / 1e3) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": ncu_traffic(name, precision, kname), "kernel": kname,
            "algorithmic_bytes_per_launch": k_amount / max(k_launch, 1),
            "ms_per_launch": k_ms / max(k_launch, 1), "step_time_share": shares, "peak_source": which,
            "model": "16 B/node-update fp32 (32 fp64) + 4*nnz + 4*(n+1) CSR bytes per iteration (SURVEY 8d); "
                     "achieved = that / CUDA-event time of the kernel's launches on the solver stream. "
                     "Every node-update is computed; K1s stores row slabs that sit on the box corners as their "
                     "sign codes (x = +-1 exactly), so the measured DRAM traffic (traffic) is below this model "
                     "(DESIGN.md 4.1)" if kname == "k_stream" else
                     "16 B/node-update fp32 (32 fp64) + 4*nnz + 4*(n+1) CSR bytes per iteration (SURVEY 8d); "
                     "achieved = that / CUDA-event time of the kernel's launches on the solver stream"}


def run_b200(args):
    import torch
    import torch.distributed as dist

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
    arm = Arm(world, rank, local, comm)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")

    sampler = ClockSampler(local) if rank == 0 else None
    main = measure(arm, args.config, args.precision, args.steps, args.warmup, flush, with_e2e=True)
    clocks = sampler.stop() if sampler else None

    extras = []
    if world == 1 and args.extras and args.config == DEFAULT_CONFIG:
        # (config, precision, steps, warm-up, host_init): the fp64 line runs the library's default
        # bit-exact mode (glibc normals drawn on the host, threaded over members)
        plan = [("c2", "fp32", 3, 3, 0), ("c3", "fp32", 3, 3, 0), ("c5", "fp32", 1, 1, 0), ("c4", "fp64", 2, 3, -1)]
        for name, prec, steps, warm, hinit in plan:
            t0 = time.perf_counter()
            try:
                r = measure(arm, name, prec, steps, warm, flush, with_e2e=False, host_init=hinit)
                extras.append({"config_id": name, "precision": prec, "steps": steps, "warmup": warm,
                               "init": "host glibc normals (bit-exact mode)" if hinit else "device normals",
                               "workload": WORKLOADS[name]["desc"], "value": r["value"], "unit": UNIT,
                               "ms_per_step": r["ms_per_step"], "best_cut": r["best_cut"], "dtype": r["dtype"],
                               "roofline_frac": r["roofline"]["frac"], "roofline": r["roofline"],
                               "wall_s": round(time.perf_counter() - t0, 1)})
            except Exception as e:  # noqa: BLE001
                extras.append({"config_id": name, "precision": prec, "error": str(e)[:300]})
            torch.cuda.empty_cache()

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                rg = reference_graph(args.config)
                T, reps = ref_sample(args.config)
                thr = os.cpu_count() or 1
                u, asc, sec, _ = cpu_reference_step(rg, args.config, 1, T, reps, thr)
                cpu = {"value": u / asc, "unit": UNIT, "cores": thr, "kind": "reference",
                       "sample": f"unmodified reference solve (oracle/_ref) of the same graph/config with T={T} "
                                 f"instead of 500" + (f", {reps} solves" if reps > 1 else "") +
                                 f", {thr} host threads; node-updates / StageTimes.ascent_s ({asc:.1f} s of "
                                 f"{sec:.1f} s solve wall)"}
                cpu["value_1_thread"], cpu["sample_1_thread"] = cpu_single_thread(rg)
            except Exception as e:  # noqa: BLE001
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}
        cfgd = config_dict(args.config, world, args.precision)
        cfgd["timing"] = "CUDA events on the solver stream around each whole solve, sum over steps, max over ranks"
        line = {
            "metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": main["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": main["dtype"], "data": "synthetic",
            "best_cut": main["best_cut"], "config": cfgd, "roofline": main["roofline"], "e2e": main["e2e"],
            "gpu_launches": main["gpu_launches"], "clocks": clocks, "cpu_baseline": cpu,
            "node_updates_per_step": main["node_updates_per_step"],
            "graph": {"nodes": main["graph_nodes"], "edges": main["graph_edges"]},
        }
        if extras:
            line["extra_configs"] = extras
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", dest="extras", action="store_false")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: launch the ranks ourselves
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
               *sys.argv[1:]]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
