"""GPU bench harness (bench_harness.py) vs the reference's benchmark families
(qcflow/bench.py:53-86): identical circuits for identical (family, n, depth, seed), the
reference's config validation, and -- on the GPU -- fused and unfused cells that agree
with each other and with the reference amplitudes."""

import json
import os

import numpy as np
import pytest

from paper_2003_02989_b200 import bench_harness as bh
from paper_2003_02989_b200.circuit import from_json, to_json

HERE = os.path.dirname(os.path.abspath(__file__))


def _cases():
    with open(os.path.join(HERE, "golden", "bench_families.json")) as f:
        return json.load(f)


def _gen(case):
    if case["family"] == "random_dense":
        return bh.gen_random_dense(case["n"], case["depth"], case["seed"])
    return bh.gen_structured(case["n"], case["depth"], 4, case["seed"])


def test_families_reproduce_reference_circuits():
    for case in _cases():
        assert bh._derive_seed(0, case["n"], case["index"]) == case["seed"]
        mine = json.loads(to_json(_gen(case)))
        ref = json.loads(case["circuit"])
        assert mine == ref


def test_config_validation_and_csv():
    with pytest.raises(ValueError):
        bh.BenchConfig(num_circuits=3, batch_size=2)
    with pytest.raises(ValueError):
        bh.BenchConfig(family="nope")
    with pytest.raises(ValueError):
        bh.gen_structured(6, 2, 4)
    rec = bh.BenchRecord(6, "random_dense", True, 30, 12, 0.5, "1.000000/0.5/0.1")
    assert bh.records_to_csv([rec]).splitlines() == [bh.CSV_HEADER, "6,random_dense,1,30,12,0.500000,1.000000/0.5/0.1"]


@pytest.mark.gpu
def test_gpu_cells_fused_unfused_and_reference_states(cuda):
    from paper_2003_02989_b200.sim import simulate_batch
    from paper_2003_02989_b200 import planner as pl

    for case in _cases():
        c = from_json(case["circuit"])
        ref = np.array(case["re"]) + 1j * np.array(case["im"])
        st = simulate_batch([c]).cpu().numpy()[0]
        np.testing.assert_allclose(st, ref, atol=1e-5)
        pl.FUSION_ENABLED = False
        try:
            st2 = simulate_batch([c]).cpu().numpy()[0]
        finally:
            pl.FUSION_ENABLED = True
        np.testing.assert_allclose(st2, ref, atol=1e-5)
    recs = bh.run_bench(bh.BenchConfig(n_qubits=(10, 12), depth=6, num_circuits=4, batch_size=2))
    assert [(r.n_qubits, r.fused) for r in recs] == [(10, True), (10, False), (12, True), (12, False)]
    for a, b in zip(recs[0::2], recs[1::2]):
        fa = [float(x) for x in a.amplitude_checksum.split("/")]
        fb = [float(x) for x in b.amplitude_checksum.split("/")]
        np.testing.assert_allclose(fa, fb, atol=2e-5)
        assert fa[0] == pytest.approx(4.0, abs=1e-4)   # four unit-norm states
        assert a.fused_gate_count < a.raw_gate_count == b.fused_gate_count
