"""Per-pass device times of the plan-specialised kernels for a BASELINE config (CUDA events
around every pass launch of one execute(); median over repetitions).

  python tools/pass_times.py cfg3 [--reps 5]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

os.environ.setdefault("QF_GRAPH", "0")  # events around each launch; a graph replay hides them

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2003_02989_b200 import jit as J  # noqa: E402
from paper_2003_02989_b200 import workloads as wl  # noqa: E402
from paper_2003_02989_b200.circuit import Circuit, circuit_symbols  # noqa: E402
from paper_2003_02989_b200.engine import ENGINE  # noqa: E402

REC = []
_run, _run_ckpt = J.JitProgram.run, J.JitProgram.run_ckpt


def _timed(self, launch, p):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    launch()
    e1.record()
    REC.append(("a" if self.prog.adjoint else "f", p, e0, e1))


def run(self, rows, *a, first=0, last=None, **k):
    last = self.n if last is None else last
    for p in range(first, last):
        _timed(self, lambda: _run(self, rows, *a, first=p, last=p + 1, **k), p)


def run_ckpt(self, *a, which=None, **k):
    for p in (range(self.n) if which is None else which):
        _timed(self, lambda: _run_ckpt(self, *a, which=[p], **k), p)


J.JitProgram.run, J.JitProgram.run_ckpt = run, run_ckpt
_turn_run = J.TurnKernel.run


def turn_run(self, *a, **k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _turn_run(self, *a, **k)
    e1.record()
    REC.append(("t", 0, e0, e1))


J.TurnKernel.run = turn_run


def bound_for(cfg):
    if cfg == "cfg1":
        circ = wl.hea_circuit(10, 4)
        syms = circuit_symbols(circ)
        return ENGINE.bind([circ] * 1024, syms, [wl.z_sum(10)], want_grad=True), \
            torch.as_tensor(wl.hea_params(1024)).cuda()
    if cfg == "cfg2":
        circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20))
        syms = circuit_symbols(circ)
        return ENGINE.bind([circ] * 256, syms, [cost], want_grad=True), torch.as_tensor(wl.qaoa_params(256, 4)).cuda()
    if cfg == "cfg3":
        from paper_2003_02989_b200 import gates as G
        phis, _, params = wl.qcnn_data(4096, 16)
        model = wl.qcnn_model(16)
        circs = [Circuit(16, list(wl.qcnn_data_circuit(p).gates) + list(model.gates)) for p in phis]
        obs = [G.PauliSum([G.PauliString(1.0, {15: "Z"})])]
        return ENGINE.bind(circs, circuit_symbols(model), obs, want_grad=True), torch.as_tensor(params).cuda()
    raise SystemExit(f"unknown config {cfg}")


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 5
    b, th = bound_for(cfg)
    for _ in range(2):
        b.execute(th, want_grad=True)
    torch.cuda.synchronize()
    samples = {}
    for _ in range(reps):
        REC.clear()
        b.execute(th, want_grad=True)
        torch.cuda.synchronize()
        for kind, p, e0, e1 in REC:
            samples.setdefault((kind, p), []).append(e0.elapsed_time(e1))
    fw = [round(float(np.median(samples[("f", p)])), 4) for p in range(len(b.plan.fwd.prog.passes))
          if ("f", p) in samples]
    ad = [round(float(np.median(samples[("a", p)])), 4) for p in range(len(b.plan.adj.prog.passes))
          if ("a", p) in samples]
    turn = round(float(np.median(samples[("t", 0)])), 4) if ("t", 0) in samples else None
    print(json.dumps({"config": cfg, "fwd_ms": fw, "adj_ms": ad, "turn_ms": turn, "fwd_total": round(sum(fw), 3),
                      "adj_total": round(sum(ad), 3), "ckpt": bool(b.plan.extra.get("ckpt")),
                      "geometry": [b.plan.fwd.prog.L, b.plan.fwd.prog.R, b.plan.adj.prog.L, b.plan.adj.prog.R]}))


if __name__ == "__main__":
    main()
