"""Generate tests/golden/* from the UNMODIFIED reference (oracle/_ref).

    make -C oracle ref && python tests/golden/make_golden.py

Everything here is produced by the reference's own code paths (Graph ctor,
generate_er, gaussian_batch, lifted_init_mean, ascend, cut_value, pquco / pluco /
pdeco / solve_per_component) through oracle/ref_shim.cpp.  The fixtures are small
enough to commit; the GPU box never needs /root/reference.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ascent_cases():
    """ascend() states after fixed horizons, fp64 bits."""
    arrays, meta = {}, []
    specs = [
        # name, graph, l, B, alpha, mu, horizons, early_exit
        ("er60", ("er", 60, 0.1, 3), 1, 6, 0.05, 0.9, [1, 5, 20, 100], False),
        ("er60_lift", ("er", 60, 0.1, 3), 2, 4, 0.05, 0.9, [1, 5, 20, 100], False),
        ("er60_l3", ("er", 60, 0.1, 3), 3, 3, 0.02, 0.5, [7, 40], False),
        ("er60_ee", ("er", 60, 0.1, 3), 1, 6, 0.2, 0.9, [400], True),
        ("er200", ("er", 200, 0.05, 11), 1, 33, 0.01, 0.9, [3, 50], False),
        ("er200_lift_ee", ("er", 200, 0.05, 11), 2, 17, 0.02, 0.0, [300], True),
    ]
    for name, gs, l, B, alpha, mu, horizons, ee in specs:
        rg = O.RefGraph.er(*gs[1:])
        g = rg.csr()
        key = O.split(7, 0x6261, len(meta))
        mean_key = O.split(5, 0x696E, len(meta))
        mean = np.zeros(g.n * l)
        O.ref.ref_lifted_init_mean(rg.h, 1, 0.2, l, mean_key, O._ptr(mean))
        mean /= 1e4
        x0 = np.zeros(B * l * g.n)
        O.ref.ref_gaussian_batch(O._ptr(mean), g.n, l, 0.8e-8, B, key, 1, O._ptr(x0))
        arrays[f"{name}/off"], arrays[f"{name}/adj"] = g.off, g.adj
        arrays[f"{name}/x0"] = x0
        for T in horizons:
            xt, _ = O.ref_ascend(rg, x0, l, B, alpha, T, mu, ee)
            arrays[f"{name}/x{T}"] = xt
        meta.append(dict(name=name, n=g.n, l=l, B=B, alpha=alpha, mu=mu, horizons=horizons,
                         early_exit=ee, gauss_key=str(key), mean_key=str(mean_key)))
    return arrays, meta


def c1_case():
    """Config 1 (ER n=800 p=0.015 seed 0, B=64, T=500): hashes + cuts."""
    rg = O.RefGraph.er(800, 0.015, 0)
    g = rg.csr()
    n, B = g.n, 64
    mean = np.zeros(n)
    O.ref.ref_lifted_init_mean(rg.h, 1, 0.2, 1, O.split(0, 0x696E, 0, 0), O._ptr(mean))
    mean /= 1e4
    key = O.split(0, 0x6261, 0)
    x0 = np.zeros(B * n)
    O.ref.ref_gaussian_batch(O._ptr(mean), n, 1, 0.8e-8, B, key, 1, O._ptr(x0))
    out = dict(n=n, m=rg.m, B=B, x0_sha=sha(x0), gauss_key=str(key), mean_sha=sha(mean))
    for T in (10, 500):
        xt, _ = O.ref_ascend(rg, x0, 1, B, 0.05, T, 0.9, False, workers=8)
        cuts = []
        for j in range(B):
            z = np.zeros(n, dtype=np.uint8)
            O.ref.ref_round_unlifted(O._ptr(xt[j * n:(j + 1) * n]), n, O._ptr(z))
            cuts.append(int(O.ref.ref_cut_value(rg.h, O._ptr(z))))
        out[f"x{T}_sha"] = sha(xt)
        out[f"cuts{T}"] = cuts
    return g, out


def solver_cases():
    cases = []
    graphs = {
        "petersen": (10, [(v, (v + 1) % 5) for v in range(5)] + [(5 + v, 5 + (v + 2) % 5) for v in range(5)]
                     + [(v, 5 + v) for v in range(5)]),
        "c5": (5, [(0, 1), (1, 2), (2, 3), (3, 4), (0, 4)]),
        "star3": (4, [(0, 1), (0, 2), (0, 3)]),
        "two_tri": (6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)]),
    }
    rgs = {k: O.RefGraph.from_edges(n, [e[0] for e in es], [e[1] for e in es]) for k, (n, es) in graphs.items()}
    rgs["er40"] = O.RefGraph.er(40, 0.15, 2)
    rgs["er120"] = O.RefGraph.er(120, 0.05, 4)
    specs = [
        ("petersen", dict(algorithm=2, batch_size=64), 0, False),
        ("c5", dict(algorithm=1, batch_size=64), 0, False),
        ("star3", dict(), 0, False),
        ("two_tri", dict(batch_size=16), 0, True),
        ("er40", dict(algorithm=0, batch_size=16, iterations=120), 9, False),
        ("er40", dict(algorithm=1, batch_size=16, iterations=120, lift_dim=3), 9, False),
        ("er40", dict(algorithm=2, batch_size=12, num_batches=2, iterations=80, has_search=1,
                      t_lower=10, t_upper=30, population_size=2, rounds=1), 9, False),
        ("er40", dict(algorithm=0, batch_size=8, num_batches=3, has_search=1, t_lower=5,
                      t_upper=40, population_size=4, rounds=2, search_refresh=1), 3, False),
        ("er120", dict(algorithm=2, batch_size=32, iterations=200, init_method=0,
                       deco_carry=1), 5, False),
        ("er120", dict(algorithm=2, batch_size=40, iterations=150, has_lifted_ascent=1,
                       l_alpha=0.01, l_iterations=90, l_momentum=0.5, l_early_exit=0,
                       resample_idi=0, scale_noise=0, eta=1e-6), 6, True),
    ]
    for gname, kw, seed, pc in specs:
        cfg = O.default_config(**kw)
        r = O.ref_solve(rgs[gname], cfg, seed, per_component=pc)
        cfgd = {f: getattr(cfg, f) for f, _ in O.Config._fields_}
        cases.append(dict(graph=gname, config=cfgd, seed=seed, per_component=pc,
                          cut=r.cut_value, batch_index=r.batch_index, member_index=r.member_index,
                          batches_run=r.batches_run, assignment=r.assignment.tolist(),
                          batch_trace=r.batch_trace, phase_trace=r.phase_trace,
                          search_trace=r.search_trace))
    csr = {k: (rg.csr().off.tolist(), rg.csr().adj.tolist()) for k, rg in rgs.items()}
    return cases, csr


def init_cases():
    rg = O.RefGraph.er(90, 0.08, 8)
    g = rg.csr()
    out = dict(off=g.off.tolist(), adj=g.adj.tolist(), cases=[])
    for key in (0, 1, 12345, 2**63 + 7):
        dui = np.zeros(g.n)
        idi = np.zeros(g.n)
        O.ref.ref_dui_init(rg.h, key, O._ptr(dui))
        O.ref.ref_idi_init(rg.h, 0.2, key, O._ptr(idi))
        lm = np.zeros(g.n * 3)
        O.ref.ref_lifted_init_mean(rg.h, 1, 0.35, 3, key, O._ptr(lm))
        out["cases"].append(dict(key=str(key), dui=dui.tolist(), idi=idi.tolist(),
                                 lifted_idi3=lm.tolist()))
    return out


def main():
    arrays, meta = ascent_cases()
    np.savez_compressed(os.path.join(OUT, "ascent_states.npz"), **arrays)
    with open(os.path.join(OUT, "ascent_states.json"), "w") as f:
        json.dump(meta, f, indent=1)
    g1, c1 = c1_case()
    with open(os.path.join(OUT, "c1_er800.json"), "w") as f:
        json.dump(c1, f, indent=1)
    cases, csr = solver_cases()
    with open(os.path.join(OUT, "solver_records.json"), "w") as f:
        json.dump(dict(graphs=csr, cases=cases), f)
    with open(os.path.join(OUT, "init_vectors.json"), "w") as f:
        json.dump(init_cases(), f)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
