"""Generate golden vectors from the REAL reference implementation (qcflow).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports qcflow from /root/reference/pkg/src (read-only) and its test helpers
(circuit_factories) from /root/reference/pkg/tests, builds circuits with the
reference API (the config recipes in paper_2003_02989_b200/workloads.py are
executed with ``lib=qcflow``), evaluates them with the reference, and writes

    tests/golden/golden.json   circuits / observables (qcflow JSON schema) + scalars
    tests/golden/golden.npz    amplitudes, gradients, bitstrings

The GPU box never reads /root/reference; tests only read these two files.
"""

from __future__ import annotations

import json
import os
import sys
import types

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def qcflow_lib():
    import qcflow
    from qcflow import circuit, gates, pauli

    ns = types.SimpleNamespace()
    for mod in (circuit, pauli, gates):
        for k in dir(mod):
            if not k.startswith("_"):
                setattr(ns, k, getattr(mod, k))
    return ns


def main():
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, REF_TESTS)
    sys.path.insert(0, ROOT)
    import qcflow
    from circuit_factories import random_concrete_circuit, random_symbolic_circuit
    from qcflow import gates as qg
    from qcflow.circuit import Circuit, Symbol, resolve, to_json
    from qcflow.fusion import fuse
    from qcflow.gradients import GradRequest, finite_difference_grad, parameter_shift_grad
    from qcflow.pauli import PauliString, PauliSum, pauli_sum_to_obj
    from qcflow.rng import derive_seed
    from qcflow.sim import batch_execute, expectation, sample, sampled_expectation, simulate

    from paper_2003_02989_b200 import workloads as wl

    L = qcflow_lib()
    meta: dict = {"reference": "qcflow " + qcflow.__version__, "numpy": np.__version__, "cases": {}}
    arrays: dict = {}

    def obs_json(o):
        return json.dumps(pauli_sum_to_obj(o if isinstance(o, PauliSum) else PauliSum([o])))

    def rand_obs(rng, n, k=4):
        terms = [PauliString(float(rng.uniform(-1, 1)))]
        for _ in range(k):
            qs = rng.choice(n, size=int(rng.integers(1, min(3, n) + 1)), replace=False)
            terms.append(PauliString(float(rng.uniform(-2, 2)), {int(q): "XYZ"[int(rng.integers(3))] for q in qs}))
        return PauliSum(terms)

    # ---- known answers (ref test_sim.py:115-130, :198-236, :342-345) ----
    bell = Circuit(2, [qg.h(0), qg.cnot(0, 1)])
    meta["cases"]["bell"] = {"circuit": to_json(bell), "zz": expectation(simulate(bell), PauliString(1.0, {0: "Z", 1: "Z"}))}
    arrays["bell/amps"] = simulate(bell).amplitudes
    c = Circuit(1, [qg.xpow(Symbol("theta"), 0)])
    meta["cases"]["xpow_ladder"] = {"circuit": to_json(c), "rows": [[0.0], [1.0], [2.0]]}
    arrays["xpow_ladder/out"] = batch_execute([c, c, c], [[0.0], [1.0], [2.0]], [PauliString(1.0, {0: "Z"})])

    # ---- random concrete circuits: states, unfused states, fusion, expectations, samples ----
    rng = np.random.default_rng(2003)
    for i, (n, depth) in enumerate([(3, 15), (4, 20), (5, 30), (6, 40), (7, 50), (8, 60), (10, 80), (11, 60)]):
        circ = random_concrete_circuit(rng, n, depth)
        name = f"concrete{i}"
        obs = [rand_obs(rng, n) for _ in range(2)]
        st = simulate(circ)
        arrays[f"{name}/amps"] = st.amplitudes
        arrays[f"{name}/amps_unfused"] = simulate(circ, fuse_enabled=False).amplitudes
        fz = fuse(circ)
        arrays[f"{name}/fused_mats"] = np.array([np.pad(g.matrix, ((0, 4 - g.matrix.shape[0]),) * 2) for g in fz.gates])
        meta["cases"][name] = {
            "circuit": to_json(circ), "n": n,
            "observables": [obs_json(o) for o in obs],
            "expectations": [expectation(st, o) for o in obs],
            "fused_targets": [list(g.targets) for g in fz.gates],
            "sample_seed": 7 + i, "shots": 300,
            "sampled_seed": 11 + i, "shots_per_term": 400,
            "sampled_expectation": sampled_expectation(circ, obs[0], 400, 11 + i),
        }
        arrays[f"{name}/bits"] = sample(st, 300, 7 + i).bitstrings

    # ---- random symbolic circuits: PS / FD gradients, evaluation accounting ----
    for i, (n, ns, depth) in enumerate([(3, 3, 10), (4, 4, 14), (5, 5, 18), (6, 4, 24)]):
        circ = random_symbolic_circuit(rng, n, ns, depth)
        obs = rand_obs(rng, n)
        syms = circ.symbols
        b = {s: float(rng.uniform(-np.pi, np.pi)) for s in syms}
        ps = parameter_shift_grad(GradRequest(circ, obs, b))
        fd = finite_difference_grad(GradRequest(circ, obs, b))
        meta["cases"][f"symbolic{i}"] = {
            "circuit": to_json(circ), "n": n, "observable": obs_json(obs), "symbols": syms,
            "bindings": [b[s] for s in syms], "ps_evaluations": ps.evaluations,
            "expectation": expectation(simulate(resolve(circ, b)), obs),
        }
        arrays[f"symbolic{i}/ps"] = ps.gradient
        arrays[f"symbolic{i}/fd"] = fd.gradient

    # ---- config-family instances built with the shared recipes, evaluated by the reference ----
    # cfg1 HEA (n=6, 2 layers), cfg2 QAOA (n=10, p=2), cfg3 QCNN (8q model + data), cfg4/5 brickwork
    hea = wl.hea_circuit(6, 2, lib=L)
    zs6 = wl.z_sum(6, lib=L)
    th = wl.hea_params(2, 6, 2).astype(np.float64)
    cfg: dict = {"hea": {"circuit": to_json(hea), "observable": obs_json(zs6), "rows": th.tolist()}}
    arrays["hea/exp"] = batch_execute([hea, hea], th, [zs6])
    arrays["hea/ps"] = np.array([parameter_shift_grad(GradRequest(hea, zs6, dict(zip(hea.symbols, r)))).gradient for r in th])

    edges = wl.qaoa_graph(10, seed=2)
    qa, cost = wl.qaoa_circuit(10, 2, edges, lib=L)
    tq = wl.qaoa_params(2, 2).astype(np.float64)
    cfg["qaoa"] = {"circuit": to_json(qa), "observable": obs_json(cost), "rows": tq.tolist(), "edges": edges}
    arrays["qaoa/exp"] = batch_execute([qa, qa], tq, [cost])
    arrays["qaoa/ps"] = np.array([parameter_shift_grad(GradRequest(qa, cost, dict(zip(qa.symbols, r)))).gradient for r in tq])

    model = wl.qcnn_model(8, lib=L)
    phis = np.random.default_rng(3).uniform(-np.pi, np.pi, size=8).astype(np.float32)
    data = wl.qcnn_data_circuit(phis.astype(np.float64), lib=L)
    full = Circuit(8, tuple(data.gates) + tuple(model.gates))
    z7 = PauliSum([PauliString(1.0, {7: "Z"})])
    pq = np.random.default_rng(4).uniform(0, 2, size=len(full.symbols)).astype(np.float32).astype(np.float64)
    cfg["qcnn"] = {"circuit": to_json(full), "observable": obs_json(z7), "row": pq.tolist()}
    arrays["qcnn/exp"] = batch_execute([full], [pq], [z7])
    arrays["qcnn/ps"] = parameter_shift_grad(GradRequest(full, z7, dict(zip(full.symbols, pq)))).gradient

    bw = wl.brickwork_circuit(10, 6, seed=401, lib=L)
    zs10 = wl.z_sum(10, lib=L)
    st = simulate(bw)
    seed_b = derive_seed(40, 0)
    cfg["rcs"] = {"circuit": to_json(bw), "observable": obs_json(zs10), "seed": seed_b,
                  "sampled": sampled_expectation(bw, zs10, 300, seed_b)}
    arrays["rcs/amps"] = st.amplitudes
    arrays["rcs/bits"] = sample(st, 200, seed_b).bitstrings
    big = wl.brickwork_circuit(12, 4, seed=5, lib=L)
    zs12 = wl.z_sum(12, lib=L)
    cfg["big"] = {"circuit": to_json(big), "observable": obs_json(zs12), "expectation": expectation(simulate(big), zs12)}
    meta["configs"] = cfg

    # ---- numpy Philox stream (pins the device RNG): first uniforms of substream(seed, *path) ----
    from qcflow.rng import substream

    meta["philox"] = []
    for seed, path in [(0, ()), (7, ()), (123456789, (3,)), (42, (1, 2))]:
        g = substream(seed, *path)
        u = g.random(9)
        key = np.random.Philox(np.random.SeedSequence(seed, spawn_key=path)).state["state"]["key"]
        meta["philox"].append({"seed": seed, "path": list(path), "key": [int(k) for k in key],
                               "uniforms": [float(x) for x in u]})

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    print("wrote", len(meta["cases"]), "cases,", len(arrays), "arrays")


if __name__ == "__main__":
    main()
