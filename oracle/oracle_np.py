"""numpy restatement of the reference FWHT path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` and ``--impl reference``) may import this module, and only
as the checker or the timed CPU baseline; the product package
``paper_1607_01039_b200`` never imports it.

Every function restates a reference function and cites it as
``/root/reference/pkg/src/bigwht/<file>:<line>``.  The arithmetic engine is
numpy, exactly as in the reference (numpy >= 2.0; the reference pins
``numpy>=1.24`` in pkg/pyproject.toml:11 but needs ``np.bitwise_count`` from
2.0, bits.py:21).  The restatement is pinned against the reference itself by
the golden fixtures under ``tests/golden/`` (made by
``tests/golden/make_golden.py`` from an import of /root/reference in the
build container) -- see ``tests/test_oracle.py``.

The generators restate this repository's own seeded spec (DESIGN.md,
"Synthetic inputs"); the reference has no generator for those
distributions.  They are bit-identical to the CUDA generator and to
``oracle/bw_oracle.c``.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

_INT64_LIMIT = 1 << 63


class OracleOverflow(ValueError):
    """M * 2**n >= 2**63 (the reference raises OverflowBoundError)."""


# ---------------------------------------------------------------- core.py ---

def check_magnitude_bound(data: np.ndarray, log2_dim: int) -> None:
    """core.py:80-94."""
    if data.dtype != np.int64 or data.size == 0:
        return
    magnitude = max(int(data.max()), -int(data.min()))
    if magnitude << log2_dim >= _INT64_LIMIT:
        raise OracleOverflow(f"max |x| = {magnitude} with n = {log2_dim}")


def fwht_array(buf: np.ndarray) -> int:
    """core.py:97-117: in-place stage loop, stage k pairs stride 2**k."""
    assert buf.flags.c_contiguous
    n = int(buf.shape[0]).bit_length() - 1
    butterflies = 0
    for k in range(n):
        pairs = buf.reshape(-1, 2, 1 << k)
        lo = pairs[:, 0, :]
        hi = pairs[:, 1, :]
        diff = lo - hi
        lo += hi
        hi[...] = diff
        butterflies += diff.size
    return butterflies


def parity_array(values: np.ndarray) -> np.ndarray:
    """bits.py:19-21."""
    return (np.bitwise_count(values) & 1).astype(np.int64)


def wht_bruteforce(x: np.ndarray, limit: int = 14) -> np.ndarray:
    """core.py:128-144: y_i = sum_j (-1)**popcount(i & j) x_j, O(4**n)."""
    n = int(x.shape[0]).bit_length() - 1
    if n > limit:
        raise ValueError(f"n = {n} exceeds the oracle limit {limit}")
    check_magnitude_bound(x, n)
    out = np.empty_like(x)
    indices = np.arange(1 << n, dtype=np.int64)
    for i in range(1 << n):
        signs = 1 - 2 * parity_array(np.bitwise_and(np.int64(i), indices))
        out[i] = signs @ x
    return out


def inverse_wht(x: np.ndarray) -> np.ndarray:
    """core.py:147-173 for int64: forward WHT then exact division by 2**n
    (returns a new array; raises ValueError when not divisible)."""
    n = int(x.shape[0]).bit_length() - 1
    y = x.copy()
    check_magnitude_bound(y, n)
    fwht_array(y)
    if np.any(y % (1 << n) != 0):
        raise ValueError("inexact division")
    return y // (1 << n)


# ------------------------------------------------------------ parallel.py ---

def plan_parallel(n: int, p: int) -> list:
    """parallel.py:87-111: phase 0 chunks, then one (start, stride, count)
    workload list per stage k = n-p .. n-1."""
    if p < 1 or p > n - 1:
        raise ValueError(f"need 1 <= p <= n-1 (got p={p}, n={n})")
    m = 1 << p
    chunk = 1 << (n - p)
    phases = [("chunks", [(w * chunk, chunk) for w in range(m)])]
    count = 1 << (n - 1 - p)
    for k in range(n - p, n):
        loads = []
        for w in range(m):
            t = w * count
            start = ((t >> k) << (k + 1)) | (t & ((1 << k) - 1))
            loads.append((start, 1 << k, count))
        phases.append((k, loads))
    return phases


def _run_workload(buf, start, stride, count):
    """parallel.py:154-159."""
    lo = buf[start:start + count]
    hi = buf[start + stride:start + stride + count]
    diff = lo - hi
    lo += hi
    hi[:] = diff


def run_parallel(buf: np.ndarray, n: int, p: int) -> None:
    """parallel.py:162-198: 2**p pool threads, a full barrier per phase."""
    plan = plan_parallel(n, p)
    with ThreadPoolExecutor(max_workers=1 << p) as pool:
        for stage, items in plan:
            if stage == "chunks":
                futs = [pool.submit(fwht_array, buf[s:s + length]) for s, length in items]
            else:
                futs = [pool.submit(_run_workload, buf, *w) for w in items]
            for f in futs:
                f.result()


# --------------------------------------------------------------- noisy.py ---

def extract_above(data: np.ndarray, tau) -> list:
    """noisy.py:185-198 + 217-222: (index, value) with |value| >= tau,
    sorted by (-|value|, index)."""
    picked = np.nonzero(np.abs(data) >= tau)[0]
    exact = data.dtype.kind == "i"  # noisy.py:219-222: int values for int arrays, float otherwise
    hits = [(int(i), int(data[i]) if exact else float(data[i])) for i in picked.tolist()]
    hits.sort(key=lambda item: (-abs(item[1]), item[0]))
    return hits


def extract_gt_by_index(data: np.ndarray, tau: int):
    """Config semantics (BASELINE.json configs 3/5): |W| > tau, by index."""
    mag = np.abs(data.astype(np.int64)).astype(np.uint64)
    mag[data == np.iinfo(np.int64).min] = np.uint64(1 << 63)
    idx = np.nonzero(mag > np.uint64(tau))[0].astype(np.int64)
    return idx, data[idx].astype(np.int64)


# ------------------------------------------------------------ subspace.py ---

def row_masks(rows: np.ndarray) -> np.ndarray:
    """subspace.py:55-59."""
    d_in = rows.shape[1]
    weights = np.int64(1) << np.arange(d_in, dtype=np.int64)
    return (rows.astype(np.int64) * weights).sum(axis=1)


def column_masks(rows: np.ndarray) -> np.ndarray:
    """subspace.py:61-65."""
    d_out = rows.shape[0]
    weights = np.int64(1) << np.arange(d_out, dtype=np.int64)
    return (rows.astype(np.int64).T * weights).sum(axis=1)


def row_space(rows: np.ndarray) -> np.ndarray:
    """subspace.py:136-147: entry i' = XOR of the rows selected by i'."""
    masks = row_masks(rows)
    d_out = rows.shape[0]
    out = np.zeros(1 << d_out, dtype=np.int64)
    for r in range(d_out):
        size = 1 << r
        out[size:2 * size] = out[:size] ^ masks[r]
    return out


def apply_map_array(rows: np.ndarray, indices: np.ndarray) -> np.ndarray:
    """subspace.py:116-121."""
    out = np.zeros(indices.shape, dtype=np.int64)
    for r, mask in enumerate(row_masks(rows).tolist()):
        out |= parity_array(indices & np.int64(mask)) << r
    return out


def fold(x: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """subspace.py:150-161: x'[L.j] += x[j]."""
    d_out, d_in = rows.shape
    out = np.zeros(1 << d_out, dtype=x.dtype)
    np.add.at(out, apply_map_array(rows, np.arange(1 << d_in, dtype=np.int64)), x)
    return out


def gf2_rank(matrix: np.ndarray) -> int:
    """subspace.py:68-89."""
    work = (np.asarray(matrix, dtype=np.uint8) % 2).copy()
    n_rows, n_cols = work.shape
    rank = 0
    for col in range(n_cols):
        pivot = -1
        for row in range(rank, n_rows):
            if work[row, col]:
                pivot = row
                break
        if pivot < 0:
            continue
        if pivot != rank:
            work[[rank, pivot]] = work[[pivot, rank]]
        for row in range(rank + 1, n_rows):
            if work[row, col]:
                work[row] ^= work[rank]
        rank += 1
        if rank == n_rows:
            break
    return rank


def random_full_rank(d_in: int, d_out: int, seed) -> np.ndarray:
    """subspace.py:92-105 (same rng draws, so the same matrix)."""
    rng = np.random.default_rng(seed)
    while True:
        candidate = rng.integers(0, 2, size=(d_out, d_in), dtype=np.uint8)
        if gf2_rank(candidate) == d_out:
            return candidate


# ------------------------------------------------------------- generators ---

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def hash64(seed: int, i: np.ndarray) -> np.ndarray:
    """h(seed, i) = fmix64(i * 0x9E3779B97F4A7C15 ^ seed) (SplitMix64
    finalizer), all mod 2**64."""
    with np.errstate(over="ignore"):
        z = (np.asarray(i, dtype=np.uint64) * _GOLD) ^ np.uint64(seed)
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return z


def gen(kind: int, seed: int, params, base: int, count: int) -> np.ndarray:
    """Values of indices base .. base+count-1 (kinds as include/bigwht_b200.h)."""
    i = np.arange(base, base + count, dtype=np.uint64)
    if kind == 1:
        return 1 - 2 * (hash64(seed, i) & np.uint64(1)).astype(np.int64)
    if kind == 2:
        a = int(params[0])
        return (hash64(seed, i) % np.uint64(2 * a + 1)).astype(np.int64) - a
    if kind == 3:
        k = int(params[0])
        thr = np.uint64(params[1])
        x = np.zeros(count, dtype=np.int64)
        for m in range(k):
            mask = np.uint64(params[2 + m])
            bit = (np.bitwise_count(mask & i) & 1).astype(np.int64)
            noise = (hash64(int(params[2 + k + m]), i) < thr).astype(np.int64)
            x += 1 - 2 * (bit ^ noise)
        return x
    raise ValueError(f"unknown kind {kind}")
