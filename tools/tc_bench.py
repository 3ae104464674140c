"""Tensor-core dense 4-qubit block (csrc/qf_tc.cu) at 2^28 amplitudes: device time, HBM GB/s
(16 B per amplitude), fraction of MEASURED_PEAKS, and the FP32 work it replaces."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2003_02989_b200 import tensorcore as tc  # noqa: E402


def main():
    n, rows = 28, 1
    rng = np.random.default_rng(0)
    q, _ = np.linalg.qr(rng.normal(size=(16, 16)) + 1j * rng.normal(size=(16, 16)))
    psi = torch.randn((rows, 1 << n), dtype=torch.complex64, device="cuda")
    out = torch.empty_like(psi)
    for _ in range(3):
        tc.apply_dense4(psi, q, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        tc.apply_dense4(psi, q, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    byts = 16 * rows * (1 << n)
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        peak = 6650.0
    gbs = byts / (ms / 1e3) / 1e9
    amps = rows * (1 << n)
    print(json.dumps({"kernel": "dense4_tc_kernel (tcgen05 kind::tf32, 3xTF32)", "amplitudes": amps, "ms": round(ms, 4),
                      "achieved_gbs": round(gbs, 1), "peak_gbs": peak, "frac": round(gbs / peak, 3),
                      "tensor_tflops": round(amps * 192 * 2 / (ms / 1e3) / 1e12, 1),
                      "ffma2_equivalent_ms": round(amps * 32 / 32 * 2 / (148 * 4 * 1.965e9) * 1e3, 3),
                      "note": "a 16x16 complex block = 16 complex MACs per amplitude = 32 FFMA2; "
                              "ffma2_equivalent_ms is the FMA-pipe floor of that work on CUDA cores"}))


if __name__ == "__main__":
    main()
