"""GF(2) subspace reduction ("fold") on the GPU.

Reference: /root/reference/pkg/src/bigwht/subspace.py.  fold(x, L) sums the
time-domain samples over the preimages of a full-rank binary map L
(subspace.py:150-161), so WHT(fold(x, L))[i'] = WHT(x)[row_space(L)[i']]
(subspace.py:1-11) -- the paper's fleet-level scheme (section 4.1)
and this repository's spot check for transforms too large for a CPU.
The small host helpers (rank, random maps, masks, row space) restate
subspace.py so the maps are the reference's own (same rng draws); the
scatter-add over 2**d_in samples is the CUDA kernel.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .core import Domain, Signal, _need_cuda, _stream_handle
from .errors import BadArguments, BadDims, BadMetadata, DimMismatch


def gf2_rank(matrix) -> int:
    """subspace.py:68-89."""
    work = (np.asarray(matrix, dtype=np.uint8) % 2).copy()
    n_rows, n_cols = work.shape
    rank = 0
    for col in range(n_cols):
        rows = np.nonzero(work[rank:, col])[0]
        if rows.size == 0:
            continue
        pivot = rank + int(rows[0])
        if pivot != rank:
            work[[rank, pivot]] = work[[pivot, rank]]
        below = rank + 1 + np.nonzero(work[rank + 1:, col])[0]
        work[below] ^= work[rank]
        rank += 1
        if rank == n_rows:
            break
    return rank


def random_full_rank(d_in: int, d_out: int, seed) -> np.ndarray:
    """subspace.py:92-105: same rejection sampling, same numpy draws."""
    if d_out < 1 or d_in < d_out:
        raise BadDims(f"need 1 <= d_out <= d_in, got {d_out}, {d_in}")
    rng = np.random.default_rng(seed)
    while True:
        candidate = rng.integers(0, 2, size=(d_out, d_in), dtype=np.uint8)
        if gf2_rank(candidate) == d_out:
            return candidate


def row_masks(rows) -> list[int]:
    """subspace.py:55-59: row r as a bitmask over input bits."""
    rows = np.asarray(rows)
    return [int(sum(int(b) << c for c, b in enumerate(r))) for r in rows]


def column_masks(rows) -> list[int]:
    """subspace.py:61-65: column c as a bitmask over output bits."""
    rows = np.asarray(rows)
    return [int(sum(int(rows[r, c]) << r for r in range(rows.shape[0]))) for c in range(rows.shape[1])]


def row_space(rows) -> np.ndarray:
    """subspace.py:136-147: entry i' = XOR of the rows selected by i'."""
    masks = row_masks(rows)
    d_out = len(masks)
    out = np.zeros(1 << d_out, dtype=np.int64)
    for r in range(d_out):
        size = 1 << r
        out[size:2 * size] = out[:size] ^ masks[r]
    return out


def _check_map(rows, d_in: int):
    rows = np.asarray(rows, dtype=np.uint8)
    if rows.ndim != 2 or rows.shape[0] < 1 or rows.shape[1] < rows.shape[0] or rows.max(initial=0) > 1:
        raise BadDims("map must be a full-rank d_out x d_in binary matrix")
    if rows.shape[1] != d_in:
        raise DimMismatch(f"signal has n={d_in}, map expects d_in={rows.shape[1]}")
    if gf2_rank(rows) != rows.shape[0]:
        raise BadDims("map must have full rank over GF(2)")
    return rows


def save_map(rows, path: str) -> None:
    """The reference's map file (subspace.py:288-293): d_out lines of d_in
    '0'/'1' characters, character c = the coefficient of input bit c."""
    rows = np.asarray(rows, dtype=np.uint8)
    with open(path, "w", encoding="utf-8") as f:
        for row in rows:
            f.write("".join("1" if v else "0" for v in row.tolist()) + "\n")


def load_map(path: str) -> np.ndarray:
    """subspace.py:296-310: the rows of a map file (BadMetadata on any
    malformed row)."""

    try:
        with open(path, "r", encoding="utf-8") as f:
            lines = [line.strip() for line in f if line.strip()]
    except OSError as exc:
        raise BadMetadata(f"cannot read map file {path}: {exc}") from exc
    if not lines:
        raise BadMetadata(f"map file {path} is empty")
    width = len(lines[0])
    for line in lines:
        if len(line) != width or set(line) - {"0", "1"}:
            raise BadMetadata(f"map file {path}: bad row {line!r}")
    return np.array([[1 if ch == "1" else 0 for ch in line] for line in lines], dtype=np.uint8)


def fold(sig: Signal, rows) -> Signal:
    """x'[L.j] += x[j] (subspace.py:150-161) on the GPU; returns a new
    time-domain Signal of 2**d_out samples (numpy in -> numpy out)."""
    if sig.domain != Domain.TIME:
        raise BadArguments("fold is defined on time-domain signals")
    if not sig.is_exact:
        raise BadArguments("the device fold is implemented for int64 signals")
    rows = _check_map(rows, sig.log2_dim)
    d_out, d_in = rows.shape
    _need_cuda()
    x = sig.data if isinstance(sig.data, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(sig.data)).cuda()
    out = torch.empty(1 << d_out, dtype=torch.int64, device=x.device)
    cols = (ctypes.c_uint64 * d_in)(*column_masks(rows))
    with torch.cuda.device(x.device):
        _lib.check(_lib.lib().bw_fold_i64(x.data_ptr(), d_in, cols, d_out, out.data_ptr(), _stream_handle(x)))
    return Signal(out if isinstance(sig.data, torch.Tensor) else out.cpu().numpy(), Domain.TIME)


def fold_generated(spec, rows, device="cuda") -> torch.Tensor:
    """fold of the seeded synthetic signal ``spec`` (signals.SignalSpec)
    without materialising it -- 2**34 samples fold in well under a second."""
    rows = _check_map(rows, spec.n)
    d_out, d_in = rows.shape
    _need_cuda()
    out = torch.empty(1 << d_out, dtype=torch.int64, device=device)
    cols = (ctypes.c_uint64 * d_in)(*column_masks(rows))
    params, count = spec.params_array()
    with torch.cuda.device(out.device):
        _lib.check(_lib.lib().bw_fold_gen_i64(d_in, spec.kind, spec.seed, params, count, cols, d_out,
                                              out.data_ptr(), _stream_handle(out)))
    return out
