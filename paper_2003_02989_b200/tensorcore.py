"""Dense gate blocks on the tcgen05 tensor cores (prototype; csrc/qf_tc.cu).

``apply_dense4(psi, U)`` applies a 16 x 16 complex unitary to qubits 0..3 (U's row/column
index bit j = qubit j, little endian like every state here) of a [rows, 2^n] complex64 device
state with kind::tf32 MMAs and 3xTF32 error compensation.  It is the building block for moving
FP32-bound dense blocks (brickwork / QCNN passes) onto the tensor cores;
the tile-pass planner does not route ops here yet.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as nat


def b_operand(u: np.ndarray) -> np.ndarray:
    """The kernel's B image of U: [2, 32, 32] float32 (tf32 hi, lo) -- qf_dense4_tc_prepare."""
    u = np.ascontiguousarray(np.asarray(u, dtype=np.complex128).reshape(16, 16))
    if u.shape != (16, 16):
        raise ValueError("apply_dense4 needs a 16 x 16 matrix")
    buf = np.ascontiguousarray(np.stack([u.real, u.imag], -1)).reshape(-1)
    out = np.empty(2 * 32 * 32, dtype=np.float32)
    nat.check(nat.load().qf_dense4_tc_prepare(buf.ctypes.data, out.ctypes.data))
    return out.reshape(2, 32, 32)


def apply_dense4(psi: torch.Tensor, u, out: torch.Tensor | None = None) -> torch.Tensor:
    """out = (U on qubits 0..3) psi for a contiguous complex64 CUDA tensor [rows, 2^n], n >= 11."""
    if not (isinstance(psi, torch.Tensor) and psi.is_cuda and psi.dtype == torch.complex64):
        raise ValueError("apply_dense4 needs a complex64 CUDA tensor")
    psi = psi.contiguous()
    rows = psi.shape[0] if psi.ndim == 2 else 1
    dim = psi.shape[-1]
    n = dim.bit_length() - 1
    if dim != 1 << n:
        raise ValueError(f"state length {dim} is not a power of two")
    b = torch.as_tensor(b_operand(u)).to(psi.device)
    if out is None:
        out = torch.empty_like(psi)
    nat.check(nat.load().qf_dense4_tc(psi.data_ptr(), out.data_ptr(), n, rows, b.data_ptr(),
                                      torch.cuda.current_stream(psi.device).cuda_stream))
    return out
