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


def _bench(args, env_extra):
    env = dict(os.environ, QF_BENCH_DEVICE="0", MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1", **env_extra)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    import json

    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_launcher_two_ranks_on_gpu():
    """bench.py --gpus 2 starts its own two ranks (torch.distributed.run); both run the headline
    step on the GPU (gloo group, QF_BENCH_DEVICE pins them to the one device) and rank 0 prints
    the max-over-ranks line for the whole 512-row job."""
    d = _bench(["--gpus", "2", "--backend", "gloo", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-ps"], {})
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 512 and d["value"] > 0
    assert d["e2e"]["value"] > 0 and d["scaling"] == "weak"


def test_bench_big32_two_ranks_on_gpu():
    """bench.py --workload big32 at 24 qubits: 2 ranks (one global qubit, gloo all-to-all of the
    shards through host memory) give the single-rank expectation."""
    one = _bench(["--workload", "big32", "--steps", "2", "--warmup", "3"], {"QF_BIG_QUBITS": "24"})
    two = _bench(["--workload", "big32", "--gpus", "2", "--backend", "gloo", "--steps", "2", "--warmup", "3"],
                 {"QF_BIG_QUBITS": "24"})
    assert two["n_gpus"] == 2 and two["config"]["global_qubits"] == 1 and two["config"]["swaps"] >= 1
    assert two["expectation"] == pytest.approx(one["expectation"], abs=1e-5)
