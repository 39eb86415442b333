import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        p = os.path.join(GOLDEN, name)
        if name.endswith(".json"):
            with open(p) as f:
                return json.load(f)
        return np.load(p)

    return load


def oracle_config(d: dict):
    import oracle as O

    c = O.default_config()
    for k, v in d.items():
        setattr(c, k, v)
    return c


def product_config(d: dict):
    """Golden config dict (lcb_config field names) -> liftcut.SolverConfig."""
    from paper_2509_18612_b200 import liftcut as lc

    a = lc.AscentParams(d["alpha"], d["iterations"], d["momentum"], bool(d["early_exit"]))
    la = (lc.AscentParams(d["l_alpha"], d["l_iterations"], d["l_momentum"], bool(d["l_early_exit"]))
          if d["has_lifted_ascent"] else None)
    init = lc.InitConfig(lc.InitMethod(d["init_method"]), d["beta"], d["eta"], d["init_scale"],
                         d["init_seed"], bool(d["resample_idi"]), bool(d["scale_noise"]))
    search = (lc.SearchConfig(d["t_lower"], d["t_upper"], d["e_lower"], d["e_upper"],
                              d["population_size"], d["rounds"]) if d["has_search"] else None)
    return lc.SolverConfig(lc.Algorithm(d["algorithm"]), d["batch_size"], d["lift_dim"], a, la, init,
                           d["num_batches"], d["time_budget_s"] if d["time_budget_s"] > 0 else None,
                           search, d["search_refresh"], d["deco_alternations"],
                           lc.DecoCarry(d["deco_carry"]))
