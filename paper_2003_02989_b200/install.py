"""Opt-in rebinding of an installed reference package onto the GPU engine.

The reference's modules import the simulation functions by name at import time
(qcflow graph.py:36, gradients.py:33, apps/_mixture.py:16, apps/vqt.py:29,
apps/qmhl.py:29, apps/qaoa.py:21, bench.py:33, cli.py:38), so replacing
``qcflow.sim.simulate`` alone would not reroute them: :func:`install` rebinds the
attribute in every importer that has it, and returns a handle whose ``undo()``
restores the originals.
"""

from __future__ import annotations

import importlib
import sys

_SIM_NAMES = ("simulate", "expectation", "batch_execute", "sample", "sampled_expectation", "run_ops",
              "apply_matrix", "pauli_term_values", "unitary")
_IMPORTERS = ("sim", "graph", "gradients", "bench", "cli", "apps._mixture", "apps.vqt", "apps.qmhl", "apps.qaoa")


class Installation:
    def __init__(self):
        self._saved: list = []

    def _set(self, mod, name, value):
        if hasattr(mod, name):
            self._saved.append((mod, name, getattr(mod, name)))
            setattr(mod, name, value)

    def undo(self):
        for mod, name, old in reversed(self._saved):
            setattr(mod, name, old)
        self._saved.clear()


def install(package: str = "qcflow") -> Installation:
    """Route ``package``'s simulation / expectation / sampling / layer calls to the GPU."""
    from . import graph as g
    from . import sim as s

    inst = Installation()
    for sub in _IMPORTERS:
        try:
            mod = importlib.import_module(f"{package}.{sub}")
        except ImportError:
            continue
        for name in _SIM_NAMES:
            inst._set(mod, name, getattr(s, name))
        if sub == "graph":
            inst._set(mod, "quantum_forward", g.quantum_forward)
            inst._set(mod, "quantum_backward", g.quantum_backward)
    root = sys.modules.get(package)
    if root is not None:
        for name in _SIM_NAMES:
            inst._set(root, name, getattr(s, name))
    return inst
