"""K2 wave-tail split (lcb_resident.cu launch_resident): at W=1024 fp32 the columns past
the last full K=2 wave run as a K=1 launch.  Per column the arithmetic is the same
(packed f32x2 adds round per lane like scalar adds, same neighbour order), so the split
must be bit-identical to the single K=2 launch (LCB_RES_SPLIT=0)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2509_18612_b200 import LCB_FP32
from paper_2509_18612_b200 import liftcut as lc

rng = np.random.default_rng(7)
n, B, T = 3000, 1024, 30
# sparse random graph plus a few hubs (heavy rows take the 8-lane subgroup path)
u = rng.integers(0, n, 12000)
v = rng.integers(0, n, 12000)
hubs = np.repeat(np.arange(4), 400)
u = np.concatenate([u, hubs])
v = np.concatenate([v, rng.integers(4, n, hubs.size)])
keep = u != v
u, v = u[keep], v[keep]
a = np.unique(np.concatenate([np.stack([u, v], 1), np.stack([v, u], 1)]), axis=0)
off = np.zeros(n + 1, np.int64)
np.add.at(off, a[:, 0] + 1, 1)
off = np.cumsum(off)
g = lc.Graph.from_csr(n, off, a[:, 1].astype(np.uint32))
s = lc.DenseState(n, 1, B)
s.values[:] = rng.uniform(-1e-2, 1e-2, s.values.shape)
lc.ascend(g, s, lc.AscentParams(0.05, T, 0.9, sys.argv[2] == '1'), precision=LCB_FP32)
assert np.all(np.abs(s.values) <= 1.0)
print(hashlib.sha256(np.ascontiguousarray(s.values).tobytes()).hexdigest())
"""


def _run(split: str, ee: bool) -> str:
    env = dict(os.environ, LCB_RES_SPLIT=split, LCB_RESIDENT="1")
    out = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, "1" if ee else "0"], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()[-1]


@pytest.mark.gpu
@pytest.mark.parametrize("ee", [False, True])
def test_resident_wave_tail_split_bitwise(ee):
    assert _run("1", ee) == _run("0", ee)
