"""Device-resident timings of every BASELINE.json config on one GPU (not the headline
bench line -- bench.py is).  One JSON line per config with circuits/s, ms per batch,
tile passes and the algorithmic-bytes GB/s of the pass kernels.

  python tools/configs_bench.py [cfg1 cfg2 cfg3 cfg4 cfg5] [--steps K]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2003_02989_b200 import ops, workloads as wl  # noqa: E402
from paper_2003_02989_b200.circuit import circuit_symbols  # noqa: E402
from paper_2003_02989_b200.engine import ENGINE  # noqa: E402
from paper_2003_02989_b200.sampling import derive_seed, philox_key, sample_indices  # noqa: E402


def timed(fn, steps, warmup=2):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def pass_bytes(bound, grad):
    from bench import pass_bytes as pb

    tot = sum(pb(bound.plan.fwd.prog, bound.B))
    if grad:
        tot += sum(pb(bound.plan.adj.prog, bound.B))
    return tot


def report(name, B, ms, bound, grad, extra=None):
    byts = pass_bytes(bound, grad)
    line = {"config": name, "rows": B, "ms_per_batch": round(ms, 4), "circuits_per_s": round(B / (ms / 1e3), 2),
            "fwd_passes": len(bound.plan.fwd.prog.passes),
            "adj_passes": len(bound.plan.adj.prog.passes) if grad else 0,
            "pass_bytes_per_batch": byts, "gbs_incl_build_reduce": round(byts / (ms / 1e3) / 1e9, 1)}
    line.update(extra or {})
    print(json.dumps(line), flush=True)


def cfg1(steps):
    circ = wl.hea_circuit(10, 4)
    syms = circuit_symbols(circ)
    th = torch.as_tensor(wl.hea_params(1024)).cuda()
    obs = [wl.z_sum(10)]
    b = ENGINE.bind([circ] * 1024, syms, obs, want_grad=True)
    ms = timed(lambda: b.execute(th, want_grad=True), steps)
    report("cfg1_hea10_b1024_adjoint", 1024, ms, b, True)
    # the configured output: parameter-shift gradients, all 1024 x 240 shifted circuits batched
    ms = timed(lambda: ops.expectation_and_ps_gradient([circ] * 1024, syms, th, obs), 1, warmup=1)
    print(json.dumps({"config": "cfg1_hea10_b1024_parameter_shift", "rows": 1024, "ms_per_batch": round(ms, 3),
                      "circuits_per_s": round(1024 / (ms / 1e3), 1), "evaluations_per_row": 241}), flush=True)


def cfg2(steps):
    circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20))
    syms = circuit_symbols(circ)
    th = torch.as_tensor(wl.qaoa_params(256, 4)).cuda()
    b = ENGINE.bind([circ] * 256, syms, [cost], want_grad=True)
    ms = timed(lambda: b.execute(th, want_grad=True), steps)
    report("cfg2_qaoa20_p4_b256_adjoint", 256, ms, b, True)


def cfg3(steps):
    phis, _, params = wl.qcnn_data(4096, 16)
    data = [wl.qcnn_data_circuit(p) for p in phis]
    model = wl.qcnn_model(16)
    from paper_2003_02989_b200.circuit import Circuit

    circs = [Circuit(16, list(d.gates) + list(model.gates)) for d in data]
    syms = circuit_symbols(model)
    th = torch.as_tensor(params).cuda()
    from paper_2003_02989_b200 import gates as G

    obs = [G.PauliSum([G.PauliString(1.0, {15: "Z"})])]
    b = ENGINE.bind(circs, syms, obs, want_grad=True)
    ms = timed(lambda: b.execute(th, want_grad=True), steps)
    report("cfg3_qcnn16_b4096_adjoint", 4096, ms, b, True)


def cfg4(steps):
    circs = wl.rcs_circuits(64, 24, 20)
    th = torch.zeros((64, 0), device="cuda")
    b = ENGINE.bind(circs, [], [])
    keys = [philox_key(derive_seed(wl.SEED_RCS_SHOTS, i)) for i in range(64)]

    def run():
        out = b.execute(th, want_state=True, want_expect=False)
        return sample_indices(out["state"], 24, 1000, keys)

    ms = timed(run, steps)
    report("cfg4_rcs24_d20_b64_state_and_1000_shots", 64, ms, b, False)


def cfg5(steps):
    circ = wl.brickwork_circuit(32, 14, wl.SEED_BIG)
    obs = [wl.z_sum(32)]
    th = torch.zeros((1, 0), device="cuda")
    b = ENGINE.bind([circ], [], obs)
    ms = timed(lambda: b.execute(th), max(1, steps // 2), warmup=1)
    e = float(b.execute(th)["expectations"][0, 0])
    report("cfg5_brickwork32_d14_expectation_1gpu", 1, ms, b, False, {"expectation": e})


def cfg5_sharded(steps):
    """The cfg-5 sharded schedule (2/4/8 shards) emulated on one GPU: every shard's tile
    passes run here and the all-to-all is a device transpose (LoopbackExchange)."""
    from paper_2003_02989_b200 import distributed as D

    circ = wl.brickwork_circuit(32, 14, wl.SEED_BIG)
    obs = wl.z_sum(32)
    for g in (1, 2, 3):
        marks = []

        def timer(kind, k):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            marks.append((kind, ev))

        e, plan = D.run_sharded(circ, obs, g, D.LoopbackExchange(g))   # warm-up (plans, JIT)
        torch.cuda.synchronize()
        marks.clear()
        t0 = time.perf_counter()
        e, plan = D.run_sharded(circ, obs, g, D.LoopbackExchange(g), timer=timer)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        parts = [(marks[i][0], round(marks[i][1].elapsed_time(marks[i + 1][1]), 2)) for i in range(len(marks) - 1)]
        print(json.dumps({"config": f"cfg5_brickwork32_d14_sharded_g{g}_loopback_1gpu", "expectation": e,
                          "swaps": plan.swaps, "wall_s": round(wall, 3), "step_ms": parts}), flush=True)
        torch.cuda.empty_cache()


def main():
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 5
    which = [a for a in sys.argv[1:] if a.startswith("cfg")] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
    for w in which:
        try:
            globals()[w](steps)
        except Exception as e:  # keep going: one line per config
            print(json.dumps({"config": w, "error": repr(e)[:300]}), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
