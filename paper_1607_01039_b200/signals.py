"""Seeded synthetic inputs of the BASELINE.json configs, generated on the GPU.

The reference has no generator for these distributions (its noisy.py:87-121
``gen`` plants Walsh amplitudes with numpy's PCG64 stream), so the spec is
this repository's own, counter based so that any slice can be regenerated
bit-identically on the CPU (oracle/oracle_np.py ``gen``, oracle/bw_oracle.c):

    h(seed, i) = fmix64((i * 0x9E3779B97F4A7C15) ^ seed)        (SplitMix64)
    PM1       : x_i = 1 - 2 * (h(seed, i) & 1)                   configs 1, 4
    UNIFORM   : x_i = h(seed, i) mod (2A + 1) - A, A = 2^20      config 2
    NOISY     : x_i = sum_k (1 - 2 * (<s_k, i> xor [h(seed_k, i) < thr]))
                K = 1, p = 0.45 (config 3); K = 8, p = 0.48 (config 5)

Noise probabilities are integers thr = floor(p * 2^64), computed once here
and handed to both the device and the CPU restatement.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch

from . import _lib

_MASK64 = (1 << 64) - 1


def hash64(seed: int, i: int) -> int:
    """Scalar h(seed, i) (host-side parameter derivation only)."""
    z = ((i * 0x9E3779B97F4A7C15) ^ seed) & _MASK64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & _MASK64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & _MASK64
    z ^= z >> 31
    return z


@dataclass(frozen=True)
class SignalSpec:
    """One seeded synthetic signal of 2**n int64 points."""

    n: int
    kind: int
    seed: int
    params: tuple = field(default_factory=tuple)
    threshold: int | None = None  # extraction threshold tau (|W| > tau), if any
    name: str = ""

    def params_array(self):
        arr = (ctypes.c_uint64 * max(1, len(self.params)))(*[int(p) & _MASK64 for p in self.params])
        return arr, len(self.params)

    @property
    def max_abs(self) -> int:
        """Bound on |x| (used for the int64 magnitude bound)."""
        if self.kind == _lib.GEN_PM1:
            return 1
        if self.kind == _lib.GEN_UNIFORM:
            return int(self.params[0])
        return int(self.params[0])

    @property
    def masks(self) -> list[int]:
        if self.kind != _lib.GEN_NOISY_MASKS:
            return []
        k = int(self.params[0])
        return [int(m) for m in self.params[2:2 + k]]


def noise_threshold(percent: int) -> int:
    """floor(percent/100 * 2**64) as an exact integer."""
    return (percent << 64) // 100


def noisy_spec(n: int, seed: int, k: int, percent: int, tau: int | None, name: str) -> SignalSpec:
    full = (1 << n) - 1
    masks, seen = [], set()
    ctr = 0
    while len(masks) < k:
        s = hash64(seed ^ 0x5EC2E75EC2E7, ctr) & full
        ctr += 1
        if s and s not in seen:
            seen.add(s)
            masks.append(s)
    seeds = [hash64(seed ^ 0x0153E0153E, m) for m in range(k)]
    return SignalSpec(n, _lib.GEN_NOISY_MASKS, seed, tuple([k, noise_threshold(percent)] + masks + seeds), tau, name)


def config(index: int, n: int | None = None) -> SignalSpec:
    """The BASELINE.json configs (1-based), optionally at another size n."""
    if index == 1:
        return SignalSpec(n or 20, _lib.GEN_PM1, 20, (), None, "config1_pm1")
    if index == 2:
        return SignalSpec(n or 24, _lib.GEN_UNIFORM, 24, (1 << 20,), None, "config2_uniform")
    if index == 3:
        return noisy_spec(n or 30, 30, 1, 45, 1 << 26, "config3_noisy_secret")
    if index == 4:
        return SignalSpec(n or 32, _lib.GEN_PM1, 32, (), None, "config4_pm1")
    if index == 5:
        return noisy_spec(n or 34, 34, 8, 48, 1 << 29, "config5_noisy_8masks")
    raise ValueError(f"no config {index}")


def generate(spec: SignalSpec, out: torch.Tensor, base: int = 0) -> torch.Tensor:
    """Fill ``out`` (CUDA int64) with indices base .. base+len(out)-1 of the
    signal, on the device (kernel K4)."""
    if not out.is_cuda or out.dtype != torch.int64 or not out.is_contiguous():
        raise ValueError("generate() needs a contiguous CUDA int64 tensor")
    arr, count = spec.params_array()
    with torch.cuda.device(out.device):
        _lib.check(_lib.lib().bw_gen_range_i64(
            out.data_ptr(), base, out.numel(), spec.kind, spec.seed, arr, count,
            torch.cuda.current_stream(out.device).cuda_stream))
    return out


def make(spec: SignalSpec, device="cuda") -> torch.Tensor:
    out = torch.empty(1 << spec.n, dtype=torch.int64, device=device)
    return generate(spec, out)
