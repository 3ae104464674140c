"""CPU executor for distributed.run_sharded backed by the oracle (test infrastructure only):
applies each rank's local circuit to its shard with the NumPy restatement of the reference."""

import numpy as np
import torch

from oracle import qcflow_port as orc


class OracleExecutor:
    def zeros(self, rows, dim):
        return torch.zeros((rows, dim), dtype=torch.complex128)

    def apply(self, circuits, names, values, psi, observables=None):
        vals = []
        for r, c in enumerate(circuits):
            bind = dict(zip(names, np.asarray(values[r], dtype=np.float64)))
            amps = psi[r].numpy().astype(np.complex128)
            amps = orc.run_ops(amps, orc.resolved_ops(c, bind), c.num_qubits, True)
            psi[r] = torch.from_numpy(amps)
            if observables is not None:
                e = 0.0
                for t in observables[r].terms:
                    if not t.factors:
                        e += t.coefficient * float(np.vdot(amps, amps).real)
                    else:
                        e += t.coefficient * float(orc.pauli_term_values(amps, t, c.num_qubits))
                vals.append(e)
        return psi, (torch.tensor(vals, dtype=torch.float64) if observables is not None else None)
