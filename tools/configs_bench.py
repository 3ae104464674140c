"""Every BASELINE.json config on one GPU, next to the reference CPU path timed on this
host's cores in the same run (not the headline bench line -- bench.py is).

One JSON line per config:
  gpu        device-resident timing (CUDA events): ms per batch, circuits/s
  roofline   algorithmic HBM bytes of the tile passes (SURVEY 8(d) rule, bench.pass_bytes)
             per batch / batch time, fraction of MEASURED_PEAKS.json hbm_gbs
  cpu        the reference algorithm (oracle port of qcflow's CPU path, test infrastructure)
             on a bounded sample: single-threaded processes on every host core; the sample
             is stated in the line
  ratio      gpu circuits/s / cpu circuits/s

  python tools/configs_bench.py [cfg1 cfg2 cfg3 cfg4 cfg5 cfg5_cpu28] [--steps K] [--no-cpu]

cfg5_cpu28 times the reference path on the cfg5 family at 28 qubits (the size the north star
names for the CPU reference; ~20 min single-threaded) and the GPU on the same circuit.
"""
import json
import os
import sys
import time

for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def _peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def timed(fn, steps, warmup=2):
    import torch

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

    ckpt = bool(bound.plan.extra.get("ckpt")) and grad
    fb = pb(bound.plan.fwd.prog, bound.B)
    tot = sum(fb)
    if grad:
        ab = pb(bound.plan.adj.prog, bound.B, ckpt=ckpt)
        tot += sum(ab)
        if ckpt and bound._turn() is not None:
            # the turn kernel (bench.py): forward's last + backward's first pass in one launch,
            # reading psi and writing lambda (16 B per amplitude) instead of both passes' bytes
            tot += 16 * (1 << bound.plan.fwd.prog.n) * bound.B - fb[-1] - ab[0]
    return tot


# ---------------------------------------------------------------------------
# CPU legs: the reference algorithm (oracle port) in single-threaded processes
# ---------------------------------------------------------------------------


def _cpu_job(args):
    """One unit of reference work in a worker process; returns seconds."""
    kind, i = args
    from oracle import qcflow_port as orc
    from paper_2003_02989_b200 import workloads as wl

    t0 = time.perf_counter()
    if kind == "cfg1_ps":                    # one parameter-shift row, 10q (gradients.py:158-165)
        circ = wl.hea_circuit(10, 4)
        from paper_2003_02989_b200.circuit import circuit_symbols

        th = wl.hea_params(1024)[i % 1024].astype(np.float64)
        bind = dict(zip(circuit_symbols(circ), th))
        orc.expectation(orc.simulate_amps(circ, bind), wl.z_sum(10), 10)
        orc.parameter_shift_grad(circ, wl.z_sum(10), bind)
    elif kind == "cfg3_eval":                # one fused 16q simulate + expectation (a PS evaluation)
        from paper_2003_02989_b200.circuit import Circuit, circuit_symbols
        from paper_2003_02989_b200.pauli import PauliString, PauliSum

        phis, _, params = wl.qcnn_data(4096, 16)
        model = wl.qcnn_model(16)
        circ = Circuit(16, list(wl.qcnn_data_circuit(phis[i % 4096]).gates) + list(model.gates))
        bind = dict(zip(circuit_symbols(model), params[i % 4096].astype(np.float64)))
        orc.expectation(orc.simulate_amps(circ, bind), PauliSum([PauliString(1.0, {15: "Z"})]), 16)
    elif kind == "cfg4_circuit":             # one 24q circuit: simulate + 1000-shot sample
        from paper_2003_02989_b200.sampling import derive_seed

        circ = wl.rcs_circuits(i + 1, 24, 20)[i]
        amps = orc.simulate_amps(circ)
        orc.sample(amps, 24, 1000, derive_seed(wl.SEED_RCS_SHOTS, i))
    elif kind == "cfg5_28":                  # the cfg5 family at 28 qubits, sum-Z
        os.environ["QCFLOW_MAX_QUBITS"] = "28"
        circ = wl.brickwork_circuit(28, 14, wl.SEED_BIG)
        orc.expectation(orc.simulate_amps(circ), wl.z_sum(28), 28)
    return time.perf_counter() - t0


def cpu_rate(kind, jobs, units_per_job, unit_name, cores=None):
    """Run ``jobs`` reference jobs on ``cores`` spawned single-threaded processes; returns
    (units/s, info)."""
    import multiprocessing as mp

    cores = cores or os.cpu_count() or 1
    ctx = mp.get_context("spawn")
    with ctx.Pool(min(cores, jobs)) as pool:
        pool.map(_cpu_noop, range(min(cores, jobs)))          # start-up, untimed
        t0 = time.perf_counter()
        per = pool.map(_cpu_job, [(kind, i) for i in range(jobs)], chunksize=1)
        wall = time.perf_counter() - t0
    return jobs * units_per_job / wall, {"cores": min(cores, jobs), "wall_s": round(wall, 2),
                                          "job_s": round(float(np.mean(per)), 3),
                                          "sample": f"{jobs} x {kind} ({units_per_job} {unit_name} each)"}


def _cpu_noop(_):
    return 0


def line(name, B, ms, byts, extra=None, cpu=None):
    peak, kind = _peak()
    gbs = byts / (ms / 1e3) / 1e9
    out = {"config": name, "rows": B, "ms_per_batch": round(ms, 4), "circuits_per_s": round(B / (ms / 1e3), 3),
           "roofline": {"bound": "hbm", "algorithmic_bytes": byts, "achieved_gbs": round(gbs, 1), "peak": peak,
                        "peak_kind": kind, "frac": round(gbs / peak, 4),
                        "note": "whole batch time (passes + builds + reductions) over the pass bytes"}}
    out.update(extra or {})
    if cpu is not None:
        out["cpu_baseline"] = cpu
        out["ratio_gpu_over_cpu"] = round(out["circuits_per_s"] / cpu["value"], 1)
    print(json.dumps(out), flush=True)


def cfg1(steps, with_cpu):
    import torch

    from paper_2003_02989_b200 import ops
    from paper_2003_02989_b200 import workloads as wl
    from paper_2003_02989_b200.circuit import circuit_symbols
    from paper_2003_02989_b200.engine import ENGINE

    circ = wl.hea_circuit(10, 4)
    syms = circuit_symbols(circ)
    th = torch.as_tensor(wl.hea_params(1024)).cuda()
    obs = [wl.z_sum(10)]
    cpu = None
    if with_cpu:
        cores = os.cpu_count() or 1
        v, info = cpu_rate("cfg1_ps", 2 * cores, 1, "row of expectation + 240 PS evaluations")
        cpu = dict(value=v, unit="circuits/s", kind="port", **info)
    # the configured output: parameter-shift gradients, all 1024 x 241 shifted circuits batched
    ms = timed(lambda: ops.expectation_and_ps_gradient(circ, syms, th, obs), steps, warmup=1)
    line("cfg1_hea10_b1024_parameter_shift", 1024, ms, 1024 * 241 * 16 * 1024, {"evaluations_per_row": 241}, cpu)
    b = ENGINE.bind([circ] * 1024, syms, obs, want_grad=True)
    ms = timed(lambda: b.execute(th, want_grad=True), steps)
    line("cfg1_hea10_b1024_adjoint", 1024, ms, pass_bytes(b, True), {"note": "L1/L2-resident (8 MiB batch)"}, cpu)


def cfg2(steps, with_cpu):
    import torch

    from paper_2003_02989_b200 import workloads as wl
    from paper_2003_02989_b200.circuit import circuit_symbols
    from paper_2003_02989_b200.engine import ENGINE

    circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20))
    syms = circuit_symbols(circ)
    th = torch.as_tensor(wl.qaoa_params(256, 4)).cuda()
    b = ENGINE.bind([circ] * 256, syms, [cost], want_grad=True)
    ms = timed(lambda: b.execute(th, want_grad=True), steps)
    line("cfg2_qaoa20_p4_b256_adjoint", 256, ms, pass_bytes(b, True),
         {"note": "the headline: bench.py carries its CPU baseline (full rows on every host core)"})


def cfg3(steps, with_cpu):
    import torch

    from paper_2003_02989_b200 import gates as G
    from paper_2003_02989_b200 import workloads as wl
    from paper_2003_02989_b200.circuit import Circuit, circuit_symbols
    from paper_2003_02989_b200.engine import ENGINE

    phis, _, params = wl.qcnn_data(4096, 16)
    model = wl.qcnn_model(16)
    circs = [Circuit(16, list(wl.qcnn_data_circuit(p).gates) + list(model.gates)) for p in phis]
    syms = circuit_symbols(model)
    th = torch.as_tensor(params).cuda()
    obs = [G.PauliSum([G.PauliString(1.0, {15: "Z"})])]
    cpu = None
    if with_cpu:
        # one row = 1 expectation + 1080 PS evaluations; time 4 evaluations per core
        cores = os.cpu_count() or 1
        v, info = cpu_rate("cfg3_eval", 4 * cores, 1.0 / 1081, "rows (one 16q evaluation = 1/1081 row)")
        cpu = dict(value=v, unit="circuits/s", kind="port", **info)
    b = ENGINE.bind(circs, syms, obs, want_grad=True)
    ms = timed(lambda: b.execute(th, want_grad=True), steps)
    line("cfg3_qcnn16_b4096_adjoint", 4096, ms, pass_bytes(b, True), None, cpu)


def cfg4(steps, with_cpu):
    import torch

    from paper_2003_02989_b200 import workloads as wl
    from paper_2003_02989_b200.engine import ENGINE
    from paper_2003_02989_b200.sampling import derive_seed, philox_key, sample_indices

    circs = wl.rcs_circuits(64, 24, 20)
    th = torch.zeros((64, 0), device="cuda")
    b = ENGINE.bind(circs, [], [], want_state=True)
    keys = [philox_key(derive_seed(wl.SEED_RCS_SHOTS, i)) for i in range(64)]
    cpu = None
    if with_cpu:
        cores = os.cpu_count() or 1
        v, info = cpu_rate("cfg4_circuit", cores, 1, "circuit: 24q simulate + 1000-shot sample")
        cpu = dict(value=v, unit="circuits/s", kind="port", **info)

    def run():
        out = b.execute(th, want_state=True, want_expect=False)
        return sample_indices(out["state"], 24, 1000, keys)

    ms = timed(run, steps)
    line("cfg4_rcs24_d20_b64_state_and_1000_shots", 64, ms, pass_bytes(b, False),
         {"fwd_passes": len(b.plan.fwd.prog.passes)}, cpu)


def cfg5(steps, with_cpu):
    import torch

    from paper_2003_02989_b200 import workloads as wl
    from paper_2003_02989_b200.engine import ENGINE

    circ = wl.brickwork_circuit(32, 14, wl.SEED_BIG)
    th = torch.zeros((1, 0), device="cuda")
    b = ENGINE.bind([circ], [], [wl.z_sum(32)])
    ms = timed(lambda: b.execute(th), max(1, steps // 2), warmup=1)
    e = float(b.execute(th)["expectations"][0, 0])
    line("cfg5_brickwork32_d14_expectation_1gpu", 1, ms, pass_bytes(b, False),
         {"expectation": e, "fwd_passes": len(b.plan.fwd.prog.passes),
          "note": "the CPU reference at 32q needs 64 GiB (c128): timed at 28q, see cfg5_cpu28"})


def cfg5_cpu28(steps, with_cpu):
    import torch

    from paper_2003_02989_b200 import workloads as wl
    from paper_2003_02989_b200.engine import ENGINE

    circ = wl.brickwork_circuit(28, 14, wl.SEED_BIG)
    th = torch.zeros((1, 0), device="cuda")
    b = ENGINE.bind([circ], [], [wl.z_sum(28)])
    ms = timed(lambda: b.execute(th), steps, warmup=1)
    cpu = None
    if with_cpu:
        v, info = cpu_rate("cfg5_28", 1, 1, "circuit: 28q simulate + sum-Z expectation", cores=1)
        cpu = dict(value=v, unit="circuits/s", kind="port", **info)
    line("cfg5_family_28q_d14_expectation_1gpu", 1, ms, pass_bytes(b, False),
         {"expectation": float(b.execute(th)["expectations"][0, 0])}, cpu)


def main():
    import torch

    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 5
    with_cpu = "--no-cpu" not in sys.argv
    which = [a for a in sys.argv[1:] if a.startswith("cfg")] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
    for w in which:
        try:
            globals()[w](steps, with_cpu)
        except Exception as e:  # keep going: one line per config
            print(json.dumps({"config": w, "error": repr(e)[:300]}), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
