"""Config-scale golden vectors from the REAL reference (qcflow), one part per process.

Run in the build container (where /root/reference exists); each part is independent
and single-threaded, so run them side by side:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_config_golden.py cfg1
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_config_golden.py cfg2     # ~30 min
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_config_golden.py cfg3
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_config_golden.py cfg4_0   # ~35 min
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_config_golden.py cfg4_1   # ~35 min
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_config_golden.py cfg4d_0  # ~2 min (per-term draws)
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_config_golden.py cfg4d_1
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_config_golden.py cfg5_28  # ~40 min, 28q
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_config_golden.py stoch

Each writes ``tests/golden/cfg/<part>.json`` (+ ``.npz`` when it has arrays).  The
circuits come from ``paper_2003_02989_b200.workloads`` executed with ``lib=qcflow``, so
the reference builds and evaluates exactly the circuits the GPU tests build with this
package.  Reference calls (file:line in /root/reference/pkg/src/qcflow):

* ``batch_execute`` (sim.py:275-294), ``simulate`` + ``expectation`` (sim.py:139-150,
  :203-213) with the qubit cap raised by ``QCFLOW_MAX_QUBITS=28`` (sim.py:27-35),
* ``sample`` (sim.py:223-227) and ``sampled_expectation`` (sim.py:245-272),
* ``parameter_shift_grad`` (gradients.py:158-165) and ``stochastic_ps_grad``
  (gradients.py:168-174).

The GPU box never reads /root/reference; tests only read the committed files.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "cfg")

# strided amplitude subsets: indices i * stride + offset, i = 0..count-1
AMP_COUNT = 4096


def amp_indices(n):
    stride = (1 << n) // AMP_COUNT
    return (np.arange(AMP_COUNT, dtype=np.int64) * stride + (np.arange(AMP_COUNT) * 7919) % stride).astype(np.int64)


def _setup():
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, REF_TESTS)
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    from make_golden import qcflow_lib

    return qcflow_lib()


def _write(part, meta, arrays=None):
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, part + ".json"), "w") as f:
        json.dump(meta, f)
    if arrays:
        np.savez_compressed(os.path.join(OUT, part + ".npz"), **arrays)
    print("wrote", part, "in", round(meta.get("seconds", 0), 1), "s", flush=True)


def part_cfg1():
    """cfg1 HEA 10q, 4 layers: 8 rows of the 1024-row batch, expectation + PS."""
    L = _setup()
    import qcflow
    from qcflow.gradients import GradRequest, parameter_shift_grad
    from qcflow.sim import batch_execute

    from paper_2003_02989_b200 import workloads as wl

    t0 = time.time()
    circ = wl.hea_circuit(10, 4, lib=L)
    obs = wl.z_sum(10, lib=L)
    rows = [0, 1, 2, 3, 511, 512, 1022, 1023]
    th = wl.hea_params(1024).astype(np.float64)[rows]
    exp = batch_execute([circ] * len(rows), th, [obs])
    ps = [parameter_shift_grad(GradRequest(circ, obs, dict(zip(circ.symbols, r)))) for r in th]
    _write("cfg1", {"reference": "qcflow " + qcflow.__version__, "rows": rows,
                    "evaluations": [p.evaluations for p in ps], "seconds": time.time() - t0},
           {"exp": exp, "ps": np.array([p.gradient for p in ps])})


def part_cfg2():
    """cfg2 QAOA 20q p=4 (the headline config): row 0 of the 256-row batch, expectation + PS."""
    L = _setup()
    import qcflow
    from qcflow.gradients import GradRequest, parameter_shift_grad
    from qcflow.sim import batch_execute

    from paper_2003_02989_b200 import workloads as wl

    t0 = time.time()
    circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20), lib=L)
    rows = [0]
    th = wl.qaoa_params(256, 4).astype(np.float64)[rows]
    exp = batch_execute([circ] * len(rows), th, [cost])
    ps = [parameter_shift_grad(GradRequest(circ, cost, dict(zip(circ.symbols, r)))) for r in th]
    _write("cfg2", {"reference": "qcflow " + qcflow.__version__, "rows": rows,
                    "evaluations": [p.evaluations for p in ps], "seconds": time.time() - t0},
           {"exp": exp, "ps": np.array([p.gradient for p in ps])})


def part_cfg3():
    """cfg3 QCNN 16q: rows 0 and 4095 (own data circuit each), expectation + PS over 72 symbols."""
    L = _setup()
    import qcflow
    from qcflow.circuit import Circuit
    from qcflow.gradients import GradRequest, parameter_shift_grad
    from qcflow.pauli import PauliString, PauliSum
    from qcflow.sim import expectation, simulate
    from qcflow.circuit import resolve

    from paper_2003_02989_b200 import workloads as wl

    t0 = time.time()
    phis, _, params = wl.qcnn_data(4096, 16)
    model = wl.qcnn_model(16, lib=L)
    obs = PauliSum([PauliString(1.0, {15: "Z"})])
    rows = [0, 4095]
    exps, grads, evs = [], [], []
    for r in rows:
        data = wl.qcnn_data_circuit(phis[r].astype(np.float64), lib=L)
        full = Circuit(16, tuple(data.gates) + tuple(model.gates))
        b = dict(zip(model.symbols, params[r].astype(np.float64)))
        exps.append(expectation(simulate(resolve(full, b)), obs))
        ps = parameter_shift_grad(GradRequest(full, obs, b))
        grads.append(ps.gradient)
        evs.append(ps.evaluations)
    _write("cfg3", {"reference": "qcflow " + qcflow.__version__, "rows": rows, "symbols": list(model.symbols),
                    "evaluations": evs, "seconds": time.time() - t0},
           {"exp": np.array(exps), "ps": np.array(grads)})


def part_cfg4(b):
    """cfg4 RCS 24q depth 20, circuit b: amplitude subset, 1000-shot sample, sampled sum-Z."""
    L = _setup()
    import qcflow
    from qcflow.rng import derive_seed
    from qcflow.sim import sample, sampled_expectation, simulate

    from paper_2003_02989_b200 import workloads as wl

    t0 = time.time()
    circ = wl.rcs_circuits(b + 1, 24, 20, lib=L)[b]
    zs = wl.z_sum(24, lib=L)
    st = simulate(circ)
    idx = amp_indices(24)
    seed_s = derive_seed(wl.SEED_RCS_SHOTS, b)
    seed_e = derive_seed(wl.SEED_RCS_SHOTS + 1, b)
    bits = sample(st, 1000, seed_s).bitstrings
    t_sim = time.time() - t0
    sexp = sampled_expectation(circ, zs, 1000, seed_e)
    _write(f"cfg4_{b}", {"reference": "qcflow " + qcflow.__version__, "circuit_index": b, "n": 24,
                         "sample_seed": seed_s, "shots": 1000, "sampled_seed": seed_e, "shots_per_term": 1000,
                         "sampled_expectation": sexp, "simulate_and_sample_seconds": t_sim,
                         "seconds": time.time() - t0},
           {"amp_idx": idx, "amps": st.amplitudes[idx], "bits": bits})


def part_cfg4d(b):
    """cfg4 circuit b, per-term draws of sampled_expectation (sim.py:245-272): sum Z needs no
    basis change, so term k draws with substream(seed_e, k) from the one simulated state --
    recorded per term (the reference function only returns their mean) and re-aggregated
    with the reference's pairwise sum to reproduce its sampled_expectation exactly."""
    L = _setup()
    import qcflow
    from qcflow.rng import derive_seed, substream
    from qcflow.sim import _draw_bits, _pairwise_sum, simulate

    from paper_2003_02989_b200 import workloads as wl

    t0 = time.time()
    circ = wl.rcs_circuits(b + 1, 24, 20, lib=L)[b]
    st = simulate(circ)
    seed_e = derive_seed(wl.SEED_RCS_SHOTS + 1, b)
    bits = np.stack([_draw_bits(st, 1000, substream(seed_e, k)) for k in range(24)])   # [24, 1000, 24]
    idx = (bits.astype(np.int64) << np.arange(24)).sum(axis=2)
    contrib = [float((1.0 - 2.0 * bits[k, :, k]).mean()) for k in range(24)]
    _write(f"cfg4d_{b}", {"reference": "qcflow " + qcflow.__version__, "circuit_index": b, "sampled_seed": seed_e,
                          "sampled_expectation_from_draws": float(_pairwise_sum(contrib)),
                          "seconds": time.time() - t0},
           {"term_idx": idx.astype(np.int32)})


def part_cfg5_28():
    """cfg5 family at 28 qubits (depth 14, SEED_BIG) with the cap override: sum-Z + amplitudes."""
    os.environ["QCFLOW_MAX_QUBITS"] = "28"
    L = _setup()
    import qcflow
    from qcflow.sim import expectation, simulate

    from paper_2003_02989_b200 import workloads as wl

    t0 = time.time()
    circ = wl.brickwork_circuit(28, 14, wl.SEED_BIG, lib=L)
    st = simulate(circ)
    t_sim = time.time() - t0
    e = expectation(st, wl.z_sum(28, lib=L))
    idx = amp_indices(28)
    _write("cfg5_28", {"reference": "qcflow " + qcflow.__version__, "n": 28, "depth": 14, "seed": wl.SEED_BIG,
                       "expectation": e, "simulate_seconds": t_sim, "seconds": time.time() - t0,
                       "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS")},
           {"amp_idx": idx, "amps": st.amplitudes[idx]})


def part_stoch():
    """stochastic_ps_grad (gradients.py:168-174) on small symbolic circuits, every sampling axis."""
    _setup()
    import qcflow
    from circuit_factories import random_symbolic_circuit
    from qcflow.circuit import to_json
    from qcflow.gradients import GradRequest, Sampled, StochasticConfig, stochastic_ps_grad
    from qcflow.pauli import PauliString, PauliSum, pauli_sum_to_obj

    t0 = time.time()
    rng = np.random.default_rng(2024)
    cases, circuits = [], []
    arrays = {}
    flags = [(False, False, False), (True, False, False), (False, True, False), (False, False, True),
             (True, True, True)]
    for i, (n, ns, depth) in enumerate([(3, 3, 10), (4, 3, 14), (5, 4, 16)]):
        circ = random_symbolic_circuit(rng, n, ns, depth)
        terms = [PauliString(0.5)]
        for _ in range(3):
            qs = rng.choice(n, size=int(rng.integers(1, 3)), replace=False)
            terms.append(PauliString(float(rng.uniform(-2, 2)), {int(q): "XYZ"[int(rng.integers(3))] for q in qs}))
        obs = PauliSum(terms)
        b = {s: float(rng.uniform(-np.pi, np.pi)) for s in circ.symbols}
        circuits.append({"circuit": to_json(circ), "observable": json.dumps(pauli_sum_to_obj(obs)),
                         "symbols": list(circ.symbols), "bindings": [b[s] for s in circ.symbols]})
        for j, (sg, sc, so) in enumerate(flags):
            for est in ("exact", "sampled"):
                cfg = StochasticConfig(sample_generator_terms=sg, sample_cost_terms=sc, sample_coordinates=so,
                                       num_samples=4, seed=100 + 10 * i + j)
                estimator = Sampled(500, 9 + i) if est == "sampled" else None
                req = GradRequest(circ, obs, b) if estimator is None else GradRequest(circ, obs, b, estimator)
                r = stochastic_ps_grad(req, cfg)
                key = f"c{i}_f{j}_{est}"
                arrays[key] = r.gradient
                cases.append({"key": key, "circuit_index": i, "flags": [sg, sc, so], "num_samples": 4, "seed": 100 + 10 * i + j,
                              "estimator": est, "shots": 500, "shot_seed": 9 + i,
                              "evaluations": r.evaluations, "degenerate": bool(r.degenerate_sampling)})
    _write("stoch", {"reference": "qcflow " + qcflow.__version__, "circuits": circuits, "cases": cases, "seconds": time.time() - t0},
           arrays)


def main():
    part = sys.argv[1]
    if part.startswith("cfg4_"):
        part_cfg4(int(part.split("_")[1]))
    elif part.startswith("cfg4d_"):
        part_cfg4d(int(part.split("_")[1]))
    else:
        globals()["part_" + part]()


if __name__ == "__main__":
    main()
