"""Command-line front end on the GPU backend: the reference CLI's simulation subcommands
(qcflow/cli.py:108-159) with the same arguments, output formats and exit codes.

    python -m paper_2003_02989_b200.cli simulate    CIRCUIT [--bindings NAME=VALUE ...] [--out F]
    python -m paper_2003_02989_b200.cli expectation CIRCUIT OBSERVABLE [--bindings ...]
    python -m paper_2003_02989_b200.cli sample      CIRCUIT --shots S --seed SEED [--bindings ...] [--out F]
    python -m paper_2003_02989_b200.cli grad        CIRCUIT OBSERVABLE [--method fd|central|ps|sps] ...

Circuit / observable files use the reference's JSON schemas (circuit.py:359-448,
pauli.py:223-244).  Exit codes (cli.py:495-499): 0 success, 1 usage error, 2 runtime
error (ValueError / KeyError / OSError / MemoryError).  The reference's ``bench`` and
``demo`` subcommands drive CPU benchmarks and training apps, outside the simulation hot
path; they keep working through ``install()``.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

from . import __version__
from .circuit import circuit_symbols, from_json, resolve
from .gradients import (CENTRAL, FORWARD, GradRequest, StochasticConfig, finite_difference_grad,
                        parameter_shift_grad, stochastic_ps_grad)
from .pauli import pauli_sum_from_obj
from .sim import expectation, sample, simulate


class _Usage(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise _Usage(f"{message}\n{self.format_usage()}")


def _pair(text: str):
    name, eq, value = text.partition("=")
    if not eq or not name:
        raise argparse.ArgumentTypeError(f"expected name=value, got {text!r}")
    try:
        return name, float(value)
    except ValueError as exc:
        raise argparse.ArgumentTypeError(f"binding {name!r} needs a numeric value") from exc


def _circuit(path):
    return from_json(Path(path).read_text())


def _observable(path):
    try:
        obj = json.loads(Path(path).read_text())
    except json.JSONDecodeError as exc:
        raise ValueError(f"invalid observable JSON in {path}: {exc}") from exc
    return pauli_sum_from_obj(obj)


def _state(args):
    return simulate(resolve(_circuit(args.circuit), dict(args.bindings or [])))


def _write(text, out):
    if out:
        Path(out).write_text(text)
    else:
        sys.stdout.write(text)


def cmd_simulate(args) -> int:
    st = _state(args)
    amps = st.amplitudes
    body = {"num_qubits": st.num_qubits, "amplitudes": [[float(a.real), float(a.imag)] for a in amps]}
    _write(json.dumps(body, indent=2) + "\n", args.out)
    return 0


def cmd_expectation(args) -> int:
    print(f"{expectation(_state(args), _observable(args.observable)):.6f}")
    return 0


def cmd_sample(args) -> int:
    bits = sample(_state(args), args.shots, args.seed).bitstrings
    counts: dict = {}
    for row in bits:
        key = "".join("1" if b else "0" for b in row)        # qubit 0 leftmost
        counts[key] = counts.get(key, 0) + 1
    _write("\n".join(["bitstring,count"] + [f"{k},{counts[k]}" for k in sorted(counts)]) + "\n", args.out)
    return 0


def cmd_grad(args) -> int:
    c = _circuit(args.circuit)
    req = GradRequest(c, _observable(args.observable), dict(args.bindings or []))
    if args.method in ("fd", "central"):
        res = finite_difference_grad(req, FORWARD if args.method == "fd" else CENTRAL, epsilon=args.epsilon)
    elif args.method == "ps":
        res = parameter_shift_grad(req)
    else:
        res = stochastic_ps_grad(req, StochasticConfig(
            sample_generator_terms=args.sample_generator_terms, sample_cost_terms=args.sample_cost_terms,
            sample_coordinates=args.sample_coordinates, num_samples=args.samples, seed=args.seed))
    for name, v in zip(circuit_symbols(c), res.gradient):
        print(f"{name} {v:.6f}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    top = _Parser(prog="paper_2003_02989_b200", description="GPU state-vector simulation (qcflow CLI subset)")
    top.add_argument("--version", action="version", version=f"paper_2003_02989_b200 {__version__}")
    sub = top.add_subparsers(dest="command", parser_class=_Parser)

    def common(p, with_obs):
        p.add_argument("circuit", help="circuit JSON file")
        if with_obs:
            p.add_argument("observable", help="observable JSON file (list of Pauli terms)")
        p.add_argument("--bindings", metavar="NAME=VALUE", type=_pair, action="append",
                       help="symbol binding (repeatable)")

    p = sub.add_parser("simulate", help="final state vector as JSON")
    common(p, False)
    p.add_argument("--out")
    p.set_defaults(func=cmd_simulate)
    p = sub.add_parser("expectation", help="exact expectation value")
    common(p, True)
    p.set_defaults(func=cmd_expectation)
    p = sub.add_parser("sample", help="measurement counts CSV")
    common(p, False)
    p.add_argument("--shots", type=int, required=True)
    p.add_argument("--seed", type=int, required=True)
    p.add_argument("--out")
    p.set_defaults(func=cmd_sample)
    p = sub.add_parser("grad", help="gradient of an expectation value")
    common(p, True)
    p.add_argument("--method", choices=("fd", "central", "ps", "sps"), default="ps")
    p.add_argument("--epsilon", type=float, default=1e-4)
    p.add_argument("--samples", type=int, default=1)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--sample-generator-terms", action="store_true")
    p.add_argument("--sample-cost-terms", action="store_true")
    p.add_argument("--sample-coordinates", action="store_true")
    p.set_defaults(func=cmd_grad)
    top.set_defaults(func=None)
    return top


def cli_main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except _Usage as exc:
        print(f"paper_2003_02989_b200: error: {exc}", file=sys.stderr)
        return 1
    except SystemExit as exc:          # --help / --version
        return int(exc.code or 0)
    if args.func is None:
        print(parser.format_usage(), file=sys.stderr, end="")
        return 1
    try:
        return args.func(args)
    except (ValueError, KeyError, OSError, MemoryError) as exc:
        print(f"paper_2003_02989_b200: error: {exc}", file=sys.stderr)
        return 2


def main() -> None:
    sys.exit(cli_main(sys.argv[1:]))


if __name__ == "__main__":
    main()
