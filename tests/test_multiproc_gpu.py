"""The CUDA engine under a real process group: two ranks (torch.distributed.run, gloo), both on
cuda:0 of the one-GPU box, each running the B200 engine on its own part of the work.

* batch sharding (bench / SURVEY 8(e) "batch"): each rank evaluates its row block with
  ``ops.expectation_and_gradient`` and ``parallel.run_sharded`` gathers the rows;
* global-qubit sharding (cfg 5 path): ``distributed.run_sharded`` with ``NcclExchange`` (its
  gloo mode stages the device shards through host memory for the all-to-all) and the engine
  executor per rank.

The ranks' kernels never wait on one another (collectives are host-side gloo calls), so two
processes may share the GPU.  Results are compared with the single-process engine."""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

BATCH_WORKER = r"""
import os, sys
sys.path.insert(0, {root!r})
import numpy as np, torch, torch.distributed as dist
dist.init_process_group("gloo")
torch.cuda.set_device(0)
from paper_2003_02989_b200 import ops, workloads as wl
from paper_2003_02989_b200.circuit import circuit_symbols
from paper_2003_02989_b200.parallel import run_sharded
circ, cost = wl.qaoa_circuit(16, 2, wl.qaoa_graph(16, seed=2))
syms = circuit_symbols(circ)
vals = wl.qaoa_params(64, 2)
def fn(rows):
    e, g = ops.expectation_and_gradient(circ, syms, rows.astype(np.float32), [cost])
    return np.concatenate([np.asarray(e, np.float64), np.asarray(g, np.float64)], axis=1)
out = run_sharded(fn, vals, 1 + len(syms))
if dist.get_rank() == 0:
    np.save(os.environ["QF_OUT"], out)
dist.destroy_process_group()
"""

GLOBAL_WORKER = r"""
import os, sys
sys.path.insert(0, {root!r})
import numpy as np, torch, torch.distributed as dist
dist.init_process_group("gloo")
torch.cuda.set_device(0)
from paper_2003_02989_b200 import distributed as D, workloads as wl
c = wl.brickwork_circuit({n}, 8, wl.SEED_BIG)
obs = wl.z_sum({n})
e, plan = D.run_sharded(c, obs, 1, D.NcclExchange(1), D.EngineExecutor())
if dist.get_rank() == 0:
    np.save(os.environ["QF_OUT"], np.array([e, plan.swaps]))
dist.destroy_process_group()
"""


def _launch(tmp_path, src, nproc=2):
    script = tmp_path / "w.py"
    script.write_text(src)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, QF_OUT=str(tmp_path / "out.npy"), MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), str(script)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(tmp_path / "out.npy")


def test_engine_batch_sharding_two_ranks(cuda, tmp_path):
    from paper_2003_02989_b200 import ops, workloads as wl
    from paper_2003_02989_b200.circuit import circuit_symbols

    got = _launch(tmp_path, BATCH_WORKER.format(root=ROOT))
    circ, cost = wl.qaoa_circuit(16, 2, wl.qaoa_graph(16, seed=2))
    syms = circuit_symbols(circ)
    e, g = ops.expectation_and_gradient(circ, syms, wl.qaoa_params(64, 2).astype(np.float32), [cost])
    want = np.concatenate([np.asarray(e, np.float64), np.asarray(g, np.float64)], axis=1)
    assert got.shape == want.shape == (64, 1 + len(syms))
    # each rank runs 32 rows x 2^16 amplitudes: the same plan-specialised kernels as 64 rows
    np.testing.assert_allclose(got, want, atol=1e-5)


def test_engine_global_qubit_sharding_two_ranks(cuda, tmp_path):
    from paper_2003_02989_b200 import ops, workloads as wl

    n = 22
    e, swaps = _launch(tmp_path, GLOBAL_WORKER.format(root=ROOT, n=n))
    c = wl.brickwork_circuit(n, 8, wl.SEED_BIG)
    want = float(ops.expectation(c, [], np.zeros((1, 0), np.float32), [wl.z_sum(n)])[0, 0])
    assert swaps >= 1
    assert e == pytest.approx(want, abs=1e-5)
