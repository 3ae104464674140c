"""Offline SASS statistics of the plan-specialised pass kernels (no GPU needed).

Generates the NVRTC sources jit.py would emit for a workload's forward/adjoint
programs, compiles them with nvcc for sm_100a, and prints registers, spills and a
static opcode histogram per pass (straight-line code: static ~= dynamic per thread).

  python tools/sass_stats.py [qaoa|rcs|qcnn|hea] [--keep DIR] [--cm]   (--cm: constant-slab adjoint variant)
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2003_02989_b200 import jit, planner as pl, workloads as wl  # noqa: E402
from paper_2003_02989_b200.circuit import circuit_symbols  # noqa: E402
from paper_2003_02989_b200.engine import _Term, _TermList, analyse_observables  # noqa: E402


def programs(name):
    if name == "qaoa":
        circ, cost = wl.qaoa_circuit(20, 4, wl.qaoa_graph(20))
    elif name == "rcs":
        circ = wl.rcs_circuits(1, 24, 20)[0]
        from paper_2003_02989_b200.pauli import PauliSum, PauliString
        cost = PauliSum([PauliString(1.0, {q: "Z"}) for q in range(24)])
    elif name == "qcnn":
        from paper_2003_02989_b200.circuit import Circuit
        from paper_2003_02989_b200.pauli import PauliSum, PauliString
        phis, _, _ = wl.qcnn_data(4, 16)
        model = wl.qcnn_model(16)
        circ = Circuit(16, list(wl.qcnn_data_circuit(phis[0]).gates) + list(model.gates))
        cost = PauliSum([PauliString(1.0, {15: "Z"})])
    elif name == "hea":
        circ = wl.hea_circuit(16, 4)
        cost = wl.z_sum(16)
    elif name == "hea10":   # cfg1's size (the parameter-shift batches run forward programs only)
        circ = wl.hea_circuit(10, 4)
        cost = wl.z_sum(10)
    else:
        raise SystemExit(f"unknown workload {name}")
    syms = circuit_symbols(circ) if name != "qcnn" else circuit_symbols(model)
    si = {s: i for i, s in enumerate(syms)}
    obs = analyse_observables([cost])
    infos = pl.analyse(circ, si)
    n = circ.num_qubits
    frame = os.environ.get("QF_FRAME", "1") != "0"
    frame_fwd = frame and pl.has_normalisable(pl.build_ops(pl.analyse(circ, si), False), pl.analyse(circ, si))
    fwd = pl.build_program(circ, infos, n, adjoint=False, observables=[_TermList(obs.sums[0])], obs_diag_ids=[0],
                           frame=frame_fwd if os.environ.get("QF_SASS_FWD_ONLY") else frame, vec=True)
    hk = [tuple(sorted(t.factors.items())) for t in obs.sums[0]]
    lam_diag = all(all(p == "Z" for _, p in k) for k in hk)
    adj = pl.build_program(circ, pl.analyse(circ, si), n, adjoint=True,
                           observables=[_TermList([_Term(dict(k), 1.0) for k in hk])], lam_diag=lam_diag,
                           frame=frame, block=os.environ.get("QF_BLOCK_ADJ", "1") not in ("0", ""), jit=True)
    return fwd, adj


def stats(src, name, keep):
    cu = os.path.join(keep, name + ".cu")
    with open(cu, "w") as f:
        f.write(jit.full_source(src))
    cub = cu.replace(".cu", ".cubin")
    r = subprocess.run(["nvcc", "-cubin", "-arch=sm_100a", "-std=c++17", "-O3", "-Xptxas", "-v", cu, "-o", cub],
                       capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr[-3000:])
    regs = re.search(r"Used (\d+) registers", r.stderr)
    spill = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", r.stderr)
    sass = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
    with open(cu.replace(".cu", ".sass"), "w") as f:
        f.write(sass)
    cnt = collections.Counter()
    for line in sass.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m:
            cnt[m.group(2)] += 1
    return int(regs.group(1)) if regs else -1, spill.groups() if spill else None, cnt


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "qaoa"
    keep = sys.argv[sys.argv.index("--keep") + 1] if "--keep" in sys.argv else "/tmp/sass"
    os.makedirs(keep, exist_ok=True)
    fwd, adj = programs(name)
    for prog, tag in ((fwd, "f"), (adj, "a")):
        srcs, names, geo = jit.generate(prog, tag, cm=("--cm" in sys.argv and prog.adjoint))
        NT = geo[0][0]
        amps = NT * (1 << prog.R)
        for s, nm in zip(srcs, names):
            regs, spill, cnt = stats(s, nm, keep)
            tot = sum(cnt.values())
            top = " ".join(f"{k}={v * NT / amps:.1f}" for k, v in cnt.most_common(10))
            print(f"{nm}: regs={regs} spill={spill} instr/amp={tot * NT / amps:.1f}  [{top}]")


if __name__ == "__main__":
    main()
