"""CPU checks of the drop-in boundary: the C-ABI library loads and exports every entry
point include/qfb200.h declares, struct layouts agree between C and ctypes, and the
multi-process batch sharding (gloo, world_size 2) reproduces the single-process result."""

import ctypes
import os
import re
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qfb200.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+(qf_\w+)\s*\(", txt, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2003_02989_b200 import _native

    lib = ctypes.CDLL(_native.LIB_PATH)
    names = _declared()
    assert len(names) >= 9
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_native.EXPORTS)


def test_struct_layouts_match_ctypes(tmp_path):
    from paper_2003_02989_b200 import _native

    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "qfb200.h"\nint main(){printf("%zu %zu %zu %zu %zu %zu\\n",'
                   'sizeof(QfProgram),sizeof(QfBuildRecipe),sizeof(QfPass),sizeof(QfStage),sizeof(QfOp),'
                   'sizeof(QfFrame));}')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    from paper_2003_02989_b200 import planner as pl

    assert got == [ctypes.sizeof(_native.QfProgram), ctypes.sizeof(_native.QfBuildRecipe),
                   4 * pl.PASS_INTS, 4 * pl.STAGE_INTS, 4 * pl.OP_INTS, ctypes.sizeof(_native.QfFrame)]
    assert ctypes.sizeof(_native.QfFrame) == 16  # engine allocates frames as [rows, 2] float64


def test_shard_rows_partition():
    from paper_2003_02989_b200.parallel import shard_rows

    for rows in (0, 1, 7, 256, 1000):
        for world in (1, 2, 3, 8):
            blocks = [shard_rows(rows, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == rows
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))


WORKER = r"""
import os, sys
sys.path.insert(0, {root!r})
import numpy as np, torch.distributed as dist
from oracle import qcflow_port as orc
from paper_2003_02989_b200 import workloads as wl
from paper_2003_02989_b200.circuit import circuit_symbols
from paper_2003_02989_b200.parallel import run_sharded
dist.init_process_group("gloo")
circ, cost = wl.qaoa_circuit(8, 2, wl.qaoa_graph(8, seed=2))
syms = circuit_symbols(circ)
vals = wl.qaoa_params(7, 2).astype(np.float64)
def fn(rows):
    return [[orc.expectation(orc.simulate_amps(circ, dict(zip(syms, r))), cost, 8)] for r in rows]
out = run_sharded(fn, vals, 1)
if dist.get_rank() == 0:
    np.save(os.environ["QF_OUT"], out)
dist.destroy_process_group()
"""


def test_gloo_world2_batch_sharding(tmp_path):
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=ROOT))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, QF_OUT=str(tmp_path / "out.npy"), MASTER_ADDR="127.0.0.1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), str(script)],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    got = np.load(tmp_path / "out.npy")
    from oracle import qcflow_port as orc
    from paper_2003_02989_b200 import workloads as wl
    from paper_2003_02989_b200.circuit import circuit_symbols

    circ, cost = wl.qaoa_circuit(8, 2, wl.qaoa_graph(8, seed=2))
    syms = circuit_symbols(circ)
    want = [[orc.expectation(orc.simulate_amps(circ, dict(zip(syms, r))), cost, 8)]
            for r in wl.qaoa_params(7, 2).astype(np.float64)]
    np.testing.assert_allclose(got, want, atol=1e-12)
