"""CPU tests (no GPU): the stochastic parameter-shift walk and accumulation against the
reference's seeded outputs (evaluated through the evaluator protocol with the CPU oracle as
the evaluator -- test infrastructure), per-topology row grouping, the bench's own multi-rank
launcher (gloo), and the C-ABI exports added this round."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import qcflow_port as orc
from paper_2003_02989_b200 import gates as G
from paper_2003_02989_b200 import gradients as gr
from paper_2003_02989_b200.circuit import Circuit, Symbol, from_json
from paper_2003_02989_b200.pauli import pauli_sum_from_obj

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


class OracleEvaluator:
    """Evaluator protocol (ref gradients.py:96-110) backed by the CPU oracle."""

    def __init__(self, estimator):
        self.estimator = estimator
        self.count = 0

    def __call__(self, circuit, observable, key=None):
        if key is None:
            key = (self.count,)
        self.count += 1
        if isinstance(self.estimator, gr.Sampled):
            seed = orc.derive_seed(self.estimator.seed, *key)
            return orc.sampled_expectation(circuit, observable, self.estimator.shots, seed)
        return orc.expectation(orc.simulate_amps(circuit), observable, circuit.num_qubits)


def test_stochastic_walk_and_accumulation_match_reference():
    """The reference's sampling walk (ref gradients.py:263-322) restated in
    gradients._stochastic_walk, accumulated in the reference's order: with an oracle
    evaluator the gradients equal qcflow's own seeded outputs (exact: 1e-10; sampled: the
    same per-evaluation substreams in complex128 -> identical draws, 1e-10)."""
    with open(os.path.join(GOLD, "cfg", "stoch.json")) as f:
        meta = json.load(f)
    arr = dict(np.load(os.path.join(GOLD, "cfg", "stoch.npz")))
    for case in meta["cases"]:
        cc = meta["circuits"][case["circuit_index"]]
        c = from_json(cc["circuit"])
        o = pauli_sum_from_obj(json.loads(cc["observable"]))
        bind = dict(zip(cc["symbols"], cc["bindings"]))
        sg, sc, so = case["flags"]
        cfg = gr.StochasticConfig(sample_generator_terms=sg, sample_cost_terms=sc, sample_coordinates=so,
                                  num_samples=case["num_samples"], seed=case["seed"])
        est = gr.Sampled(case["shots"], case["shot_seed"]) if case["estimator"] == "sampled" else gr.Exact()
        ev = OracleEvaluator(est)
        r = gr.stochastic_ps_grad(gr.GradRequest(c, o, bind, est), cfg, evaluator=ev)
        assert r.evaluations == case["evaluations"] == ev.count
        assert r.degenerate_sampling == case["degenerate"]
        np.testing.assert_allclose(r.gradient, arr[case["key"]], atol=1e-10, err_msg=case["key"])


def test_topology_groups_split_rows_by_structure():
    from paper_2003_02989_b200.ops import topology_groups

    base = [G.h(0), G.cz(0, 1)]
    rows = [Circuit(3, base + [G.rx(0.1 * (b + 1), b % 3), G.ry(Symbol("t"), 2)]) for b in range(7)]
    groups = topology_groups(rows, ["t"])
    assert sorted(map(list, groups)) == [[0, 3, 6], [1, 4], [2, 5]]
    with pytest.raises(KeyError):
        topology_groups(rows, ["other"])


def test_bench_launcher_spawns_ranks_gloo():
    """``bench.py --gpus 2`` without a torchrun environment starts 2 ranks itself (VERDICT r1
    next #4); --dry-run exercises the rank plumbing (shards, barrier, max-reduce) on gloo."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["rows_evaluated"] == line["global_batch"] == 16


def test_new_exports_declared_and_bound():
    from paper_2003_02989_b200 import _native

    hdr = open(os.path.join(ROOT, "include", "qfb200.h")).read()
    for name in ("qf_sample_multi", "qf_reduce_slots_offset"):
        assert name in _native.EXPORTS
        assert f"int {name}(" in hdr
    lib = _native.load(build_if_missing=False)
    for name in _native.EXPORTS:
        assert hasattr(lib, name)
