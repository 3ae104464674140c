"""CLI golden outputs from the REAL reference command line (qcflow/cli.py:108-159, cli_main
:487-500), run in the build container.  Writes tests/golden/cli.json: input files (circuit /
observable JSON text), argv, exit code and stdout of each invocation.  The GPU tests replay
the same argv through paper_2003_02989_b200.cli.cli_main."""

import contextlib
import io
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, REF_TESTS)
    import tempfile

    from circuit_factories import random_concrete_circuit, random_symbolic_circuit
    from qcflow import gates as qg
    from qcflow.circuit import Circuit, Symbol, to_json
    from qcflow.cli import cli_main
    from qcflow.pauli import PauliString, PauliSum, pauli_sum_to_obj

    rng = np.random.default_rng(77)
    files = {
        "bell.json": to_json(Circuit(2, [qg.h(0), qg.cnot(0, 1)])),
        "zz.json": json.dumps(pauli_sum_to_obj(PauliSum([PauliString(1.0, {0: "Z", 1: "Z"})]))),
        "rot.json": to_json(Circuit(1, [qg.rx(Symbol("theta"), 0)])),
        "z0.json": json.dumps(pauli_sum_to_obj(PauliSum([PauliString(1.0, {0: "Z"})]))),
        "rand6.json": to_json(random_concrete_circuit(rng, 6, 40)),
        "sym4.json": to_json(random_symbolic_circuit(rng, 4, 3, 16)),
        "obs4.json": json.dumps(pauli_sum_to_obj(PauliSum([PauliString(0.5), PauliString(1.2, {0: "Z", 2: "X"}),
                                                           PauliString(-0.7, {1: "Y"}), PauliString(0.4, {3: "Z"})]))),
    }
    import qcflow.circuit as qc

    syms = qc.from_json(files["sym4.json"]).symbols
    binds = []
    for s in syms:
        binds += ["--bindings", f"{s}={float(rng.uniform(-2, 2)):.6f}"]
    runs = [
        ["expectation", "bell.json", "zz.json"],
        ["simulate", "bell.json"],
        ["simulate", "rand6.json"],
        ["expectation", "rand6.json", "obs4.json"],
        ["sample", "rand6.json", "--shots", "500", "--seed", "7"],
        ["sample", "bell.json", "--shots", "64", "--seed", "3"],
        ["grad", "rot.json", "z0.json", "--method", "ps", "--bindings", "theta=0.3"],
        ["grad", "sym4.json", "obs4.json", "--method", "ps"] + binds,
        ["grad", "sym4.json", "obs4.json", "--method", "central", "--epsilon", "1e-3"] + binds,
        ["grad", "sym4.json", "obs4.json", "--method", "sps", "--samples", "3", "--seed", "5",
         "--sample-generator-terms", "--sample-coordinates"] + binds,
        ["expectation", "sym4.json", "obs4.json"],          # unresolved symbol -> exit 2
        ["sample", "rand6.json", "--shots", "5"],            # missing --seed -> usage error, exit 1
    ]
    out = {"files": files, "runs": []}
    with tempfile.TemporaryDirectory() as d:
        for name, text in files.items():
            with open(os.path.join(d, name), "w") as f:
                f.write(text)
        cwd = os.getcwd()
        os.chdir(d)
        try:
            for argv in runs:
                buf, err = io.StringIO(), io.StringIO()
                with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(err):
                    rc = cli_main(argv)
                out["runs"].append({"argv": argv, "rc": rc, "stdout": buf.getvalue()})
        finally:
            os.chdir(cwd)
    with open(os.path.join(HERE, "cli.json"), "w") as f:
        json.dump(out, f)
    print("wrote", len(out["runs"]), "CLI runs")


if __name__ == "__main__":
    main()
