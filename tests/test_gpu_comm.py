"""The NCCL exchange path on the one GPU of the box: a 1-rank communicator runs the
same ncclAllReduce calls (packed key, winner bits, error slots) on the solver stream;
results must equal the communicator-free solve.  (Multi-rank correctness of the
exchange protocol itself is tests/test_dist_cpu.py.)"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

CODE = r"""
import os, socket, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.distributed as dist
import oracle as O
from paper_2509_18612_b200 import liftcut as lc, LCB_FP64, LCB_FP32
from paper_2509_18612_b200.dist import Comm
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
comm = Comm.from_torch(0)
cg = O.generate_er(400, 0.03, 9)
g = lc.Graph.from_csr(cg.n, cg.off, cg.adj)
for prec in (LCB_FP64, LCB_FP32):
    cfg = lc.SolverConfig(algorithm=lc.Algorithm.pDECO, batch_size=40, ascent=lc.AscentParams(0.05, 120),
                          num_batches=2, search=lc.SearchConfig(10, 40, -3.0, -1.0, 4, 2))
    a = lc.pdeco(g, cfg, 3, opts=lc.RunOptions(precision=prec, host_init=0))
    b = lc.pdeco(g, cfg, 3, opts=lc.RunOptions(precision=prec, host_init=0, comm=comm, batched_search=True))
    assert a.best.cut_value == b.best.cut_value, (a.best.cut_value, b.best.cut_value)
    assert np.array_equal(a.best.assignment, b.best.assignment)
    assert [e.batch_best for e in a.batch_trace] == [e.batch_best for e in b.batch_trace]
comm.close()
dist.destroy_process_group()
print("comm ok")
"""


def test_one_rank_nccl_exchange_matches_local_solve():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", CODE], cwd=root, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "LCB_FORCE_NCCL": "1"})
    assert r.returncode == 0 and "comm ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
