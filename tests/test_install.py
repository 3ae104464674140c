"""install(): rebinding of a reference-shaped package (qcflow's importer modules bind the
simulation functions by name, ref graph.py:36, gradients.py:33, bench.py:33, cli.py:38)."""

import os
import sys

import numpy as np
import pytest

from paper_2003_02989_b200 import install as inst_mod
from paper_2003_02989_b200 import sim as our_sim

FAKE = {
    "__init__.py": "from .sim import simulate, expectation\n",
    "sim.py": "def simulate(c, fuse_enabled=True):\n    return 'cpu'\n\ndef expectation(s, o):\n    return 'cpu'\n"
              "def sample(s, shots, seed):\n    return 'cpu'\n",
    "graph.py": "from .sim import simulate, expectation\n\ndef quantum_forward(node, b):\n    return 'cpu'\n"
                "def quantum_backward(node, b, u):\n    return 'cpu'\n",
    "bench.py": "from .sim import simulate\n",
    "cli.py": "from .sim import simulate, sample\n",
}


@pytest.fixture()
def fakepkg(tmp_path, monkeypatch):
    pkg = tmp_path / "fakeqc"
    pkg.mkdir()
    for name, body in FAKE.items():
        (pkg / name).write_text(body)
    monkeypatch.syspath_prepend(str(tmp_path))
    yield "fakeqc"
    for k in [k for k in sys.modules if k == "fakeqc" or k.startswith("fakeqc.")]:
        del sys.modules[k]


def test_install_rebinds_every_importer_and_undo_restores(fakepkg):
    import importlib

    root = importlib.import_module(fakepkg)
    graph = importlib.import_module(fakepkg + ".graph")
    bench = importlib.import_module(fakepkg + ".bench")
    cli = importlib.import_module(fakepkg + ".cli")
    h = inst_mod.install(fakepkg)
    try:
        assert root.simulate is our_sim.simulate and root.sim.simulate is our_sim.simulate
        assert graph.simulate is our_sim.simulate and bench.simulate is our_sim.simulate
        assert cli.sample is our_sim.sample
        from paper_2003_02989_b200 import graph as our_graph

        assert graph.quantum_forward is our_graph.quantum_forward
        assert graph.quantum_backward is our_graph.quantum_backward
    finally:
        h.undo()
    assert root.simulate(None) == "cpu" and graph.simulate(None) == "cpu" and cli.sample(None, 1, 0) == "cpu"
    assert graph.quantum_forward(None, None) == "cpu"


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference sources not present")
def test_install_on_the_real_reference_package(monkeypatch):
    """Only in the build container: the rebinding reaches qcflow's own importers."""
    monkeypatch.syspath_prepend("/root/reference/pkg/src")
    import qcflow
    import qcflow.bench
    import qcflow.graph
    import qcflow.sim

    h = inst_mod.install("qcflow")
    try:
        assert qcflow.sim.simulate is our_sim.simulate
        assert qcflow.bench.simulate is our_sim.simulate
        assert qcflow.graph.quantum_backward is not None
    finally:
        h.undo()
    assert qcflow.sim.simulate is not our_sim.simulate


@pytest.mark.gpu
def test_installed_fake_package_runs_on_gpu(cuda, fakepkg):
    import importlib

    from oracle import qcflow_port as orc
    from paper_2003_02989_b200 import workloads as wl

    bench = importlib.import_module(fakepkg + ".bench")
    h = inst_mod.install(fakepkg)
    try:
        c = wl.brickwork_circuit(8, 4, 7)
        st = bench.simulate(c)
        np.testing.assert_allclose(st.amplitudes, orc.simulate_amps(c), atol=1e-5)
    finally:
        h.undo()
