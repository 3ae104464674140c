"""CPU oracle package -- test infrastructure only (see qcflow_port.py header)."""
