"""Shot sampling with the reference's exact draw semantics (qcflow/sim.py:216-227).

The reference draws ``Generator(Philox(SeedSequence(seed, spawn_key=path))).choice(
2^n, shots, p=|a|^2/sum)``.  numpy's ``choice`` with ``p`` is
``searchsorted(cumsum(p)/cdf[-1], random(shots), side='right')`` and ``random()`` is
``(next_uint64 >> 11) * 2^-53`` from Philox4x64-10 blocks with counters 1, 2, ...
The GPU reproduces that stream bit-for-bit (qf_sample) from the 128-bit Philox key,
which the host derives with numpy's own SeedSequence -- so the same seed gives the
same uniforms on both sides, and the same state gives the same bitstrings.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as nat


def philox_key(seed: int, *path: int) -> tuple[int, int]:
    """Key of ``substream(seed, *path)`` (ref rng.py:14-19)."""
    if seed < 0:
        raise ValueError("seed must be non-negative")
    seq = np.random.SeedSequence(int(seed), spawn_key=tuple(int(p) for p in path))
    st = np.random.Philox(seq).state["state"]
    k = st["key"]
    return int(k[0]), int(k[1])


def derive_seed(seed: int, *path: int) -> int:
    """ref rng.py:22-27."""
    if seed < 0:
        raise ValueError("seed must be non-negative")
    return int(np.random.SeedSequence(int(seed), spawn_key=tuple(int(p) for p in path)).generate_state(1, np.uint64)[0])


def sample_indices(psi: torch.Tensor, n_eff: int, shots: int, keys, stream=None, keys_per_row: int = 1):
    """psi: [B, 2^n_eff] complex64 on device; keys: [(k0, k1)] per row (``keys_per_row`` > 1:
    row-major [B, keys_per_row] keys, every key of a row drawing from that row's CDF).
    Returns (indices [B, shots] -- [B, keys_per_row, shots] when keys_per_row > 1 -- int64
    device tensor, near-boundary counts int32)."""
    if shots < 1:
        raise ValueError("shots must be >= 1")
    lib = nat.load()
    B = psi.shape[0]
    K = int(keys_per_row)
    dev = psi.device
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    kt = torch.tensor(np.array(keys, dtype=np.uint64).reshape(B * K, 2).view(np.int64), device=dev)
    nchunk = (1 << n_eff) // 1024
    scratch = torch.empty(B * (2 * nchunk + 1) + 8, dtype=torch.float64, device=dev)
    idx = torch.empty((B, K, shots) if K > 1 else (B, shots), dtype=torch.int64, device=dev)
    near = torch.zeros(B * K, dtype=torch.int32, device=dev)
    nat.check(lib.qf_sample_multi(psi.data_ptr(), n_eff, B, K, shots, kt.data_ptr(), scratch.data_ptr(),
                                  idx.data_ptr(), near.data_ptr(), stream))
    return idx, near


def bits_from_indices(idx: np.ndarray, n: int) -> np.ndarray:
    """[..., shots] indices -> [..., shots, n] uint8, column q = qubit q (ref sim.py:220)."""
    return ((idx[..., None] >> np.arange(n)) & 1).astype(np.uint8)
