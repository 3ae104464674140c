import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
os.environ["QF_JIT"] = "1"
from paper_2003_02989_b200 import workloads as wl, ops
from paper_2003_02989_b200.circuit import Circuit, circuit_symbols
from paper_2003_02989_b200.pauli import PauliString, PauliSum
from paper_2003_02989_b200.engine import ENGINE
sys.path.insert(0, "tests")
import oracle_shim  # noqa
