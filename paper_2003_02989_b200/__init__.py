"""B200-native batched state-vector simulation of parameterised quantum circuits.

A drop-in for the hot path of the reference package ``qcflow`` (a NumPy
re-implementation of TensorFlow Quantum's core, arXiv:2003.02989): the state,
expectation, sampled-expectation and sample ops and their adjoint and
parameter-shift differentiators, with the reference's call signatures, running
on hand-written sm_100a CUDA kernels through the C ABI in ``include/qfb200.h``.

Modules
  circuit / pauli / gates   host-side IR (same data model as qcflow)
  sim                       qcflow.sim-compatible functions (GPU-backed)
  gradients                 GradRequest/GradResult, Adjoint, ParameterShift, FD, stochastic PS
  graph                     batched quantum_forward / quantum_backward for layer nodes
  ops                       TFQ-style batched ops: op(circuits, symbol_names, symbol_values, operators)
  engine / planner          plan cache, fusion, tile-pass programs
  install                   rebind an installed qcflow onto this engine
"""

from .circuit import Circuit, Gate, ParamExpr, Symbol, compose, exponential_circuit, from_json, gate_matrix, \
    resolve, to_json
from .pauli import PauliString, PauliSum, identity, pauli_sum_from_obj, pauli_sum_to_obj, pauli_x, pauli_y, pauli_z
from .sampling import derive_seed, philox_key

__version__ = "0.1.0"

_LAZY = {
    "sim": ".sim", "gradients": ".gradients", "graph": ".graph", "ops": ".ops", "engine": ".engine",
    "planner": ".planner", "gates": ".gates", "workloads": ".workloads", "install": ".install",
    "cli": ".cli",
}
_LAZY_ATTRS = {
    "simulate": "sim", "expectation": "sim", "batch_execute": "sim", "sample": "sim",
    "sampled_expectation": "sim", "StateVector": "sim", "SampleBatch": "sim", "unitary": "sim",
    "GradRequest": "gradients", "GradResult": "gradients", "Exact": "gradients", "Sampled": "gradients",
    "StochasticConfig": "gradients", "Adjoint": "gradients", "ParameterShift": "gradients",
    "FiniteDifference": "gradients", "StochasticShift": "gradients", "adjoint_grad": "gradients",
    "parameter_shift_grad": "gradients", "finite_difference_grad": "gradients",
    "stochastic_ps_grad": "gradients", "quantum_forward": "graph", "quantum_backward": "graph",
}


def __getattr__(name):
    import importlib

    if name in _LAZY:
        return importlib.import_module(_LAZY[name], __name__)
    if name in _LAZY_ATTRS:
        mod = importlib.import_module("." + _LAZY_ATTRS[name], __name__)
        return getattr(mod, name)
    raise AttributeError(name)
