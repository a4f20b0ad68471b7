"""The reference's on-disk dataset format, read and written for the GPU engine.

Format (/root/reference/pkg/src/bigwht/dataset.py:1-88): a raw
little-endian array of 2**n 8-byte elements plus a JSON sidecar
``<path>.meta.json`` holding format_version (1), log2_dim, element_kind
(int64 | float64) and domain (time | walsh); the sidecar is replaced
atomically.  Payloads are memory-mapped, so the out-of-core transform and
the extraction stream them without loading them whole.  The pass-progress
marker / resume protocol of the reference's disk executor is out of scope.
"""

from __future__ import annotations

import json
import os

import numpy as np

from .errors import BadArguments, BadMetadata, PathExists, SizeMismatch

ELEMENT_BYTES = 8
FORMAT_VERSION = 1
_DTYPES = {"int64": np.dtype("<i8"), "float64": np.dtype("<f8")}
_DOMAINS = ("time", "walsh")


def sidecar_path(path: str) -> str:
    return path + ".meta.json"


def _write_sidecar(path: str, meta: dict) -> None:
    tmp = sidecar_path(path) + ".tmp"
    with open(tmp, "w", encoding="utf-8") as f:
        json.dump(meta, f, indent=2, sort_keys=True)
        f.write("\n")
        f.flush()
        os.fsync(f.fileno())
    os.replace(tmp, sidecar_path(path))


def read_meta(path: str) -> dict:
    """Validated sidecar (dataset.py:69-88 semantics)."""
    try:
        with open(sidecar_path(path), "r", encoding="utf-8") as f:
            meta = json.load(f)
    except FileNotFoundError as exc:
        raise BadMetadata(f"missing sidecar {sidecar_path(path)}") from exc
    except (OSError, json.JSONDecodeError) as exc:
        raise BadMetadata(f"unreadable sidecar {sidecar_path(path)}: {exc}") from exc
    if not isinstance(meta, dict) or meta.get("format_version") != FORMAT_VERSION:
        raise BadMetadata(f"unsupported sidecar in {sidecar_path(path)}")
    n = meta.get("log2_dim")
    if not isinstance(n, int) or n < 0:
        raise BadMetadata(f"bad log2_dim {n!r}")
    if meta.get("element_kind") not in _DTYPES:
        raise BadMetadata(f"bad element_kind {meta.get('element_kind')!r}")
    if meta.get("domain") not in _DOMAINS:
        raise BadMetadata(f"bad domain {meta.get('domain')!r}")
    try:
        size = os.path.getsize(path)
    except OSError as exc:
        raise SizeMismatch(f"payload {path} is missing: {exc}") from exc
    if size != ELEMENT_BYTES << n:
        raise SizeMismatch(f"{path} is {size} bytes, sidecar says 2**{n} elements")
    return meta


def open_memmap(path: str, mode: str = "r+") -> tuple[np.memmap, dict]:
    meta = read_meta(path)
    arr = np.memmap(path, dtype=_DTYPES[meta["element_kind"]], mode=mode, shape=(1 << meta["log2_dim"],))
    return arr, meta


def set_domain(path: str, domain: str) -> None:
    if domain not in _DOMAINS:
        raise BadArguments(f"bad domain {domain!r}")
    meta = read_meta(path)
    meta["domain"] = domain
    _write_sidecar(path, meta)


def write_signal(path: str, data: np.ndarray, domain: str = "time") -> None:
    """Create a dataset holding ``data`` (dataset.py:427-446 semantics)."""
    arr = np.asarray(data)
    kind = {np.dtype(np.int64): "int64", np.dtype(np.float64): "float64"}.get(arr.dtype)
    if kind is None:
        raise BadArguments(f"unsupported dtype {arr.dtype}")
    n = int(arr.shape[0]).bit_length() - 1
    if arr.ndim != 1 or (1 << n) != arr.shape[0]:
        raise BadArguments("length must be a power of two")
    if domain not in _DOMAINS:
        raise BadArguments(f"bad domain {domain!r}")
    if os.path.exists(path) or os.path.exists(sidecar_path(path)):
        raise PathExists(f"{path} (or its sidecar) already exists")
    arr.astype(_DTYPES[kind], copy=False).tofile(path)
    _write_sidecar(path, {"format_version": FORMAT_VERSION, "log2_dim": n, "element_kind": kind, "domain": domain})


def adopt(path: str, element_kind: str, domain: str) -> int:
    """Write a sidecar for a bare payload of 8 * 2**n bytes, inferring n
    from the file size (dataset.py:408-435 semantics).  Returns n."""
    if element_kind not in _DTYPES:
        raise BadArguments(f"bad element_kind {element_kind!r}")
    if domain not in _DOMAINS:
        raise BadArguments(f"bad domain {domain!r}")
    if os.path.exists(sidecar_path(path)):
        raise PathExists(f"{sidecar_path(path)} already exists")
    try:
        size = os.path.getsize(path)
    except OSError as exc:
        raise SizeMismatch(f"payload {path} is missing: {exc}") from exc
    count = size // ELEMENT_BYTES
    if size % ELEMENT_BYTES or count < 1 or count & (count - 1):
        raise SizeMismatch(f"{path} is {size} bytes, not 8 * 2**n; cannot infer a dimension")
    n = count.bit_length() - 1
    _write_sidecar(path, {"format_version": FORMAT_VERSION, "log2_dim": n, "element_kind": element_kind,
                          "domain": domain})
    return n


def read_signal(path: str) -> tuple[np.ndarray, str, str]:
    """(array, element_kind, domain) -- the whole payload in memory."""
    meta = read_meta(path)
    arr = np.fromfile(path, dtype=_DTYPES[meta["element_kind"]]).astype(_DTYPES[meta["element_kind"]].newbyteorder("="))
    return arr, meta["element_kind"], meta["domain"]


__all__ = ["BadMetadata", "SizeMismatch", "PathExists", "adopt", "open_memmap", "read_meta",
           "read_signal", "set_domain", "sidecar_path", "write_signal"]
