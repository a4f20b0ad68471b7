"""Command line on the GPU engine: ``python -m paper_1607_01039_b200 ...``.

Mirrors the reference CLI's commands around the transform
(/root/reference/pkg/src/bigwht/cli.py: transform mem/ext 144-219, oracle
225-257, extract 260-291, fold 477-518, the global --seed / --quiet /
--json / --force options 41-84) on the reference's dataset format: the same
options, exit codes (0 ok, 1 usage, 2 I/O, 3 validation; cli.py:561-584),
stderr diagnostics suppressed by --quiet and the ``--json``
schema-version-1 documents.  ``gen-config`` writes the seeded BASELINE.json
configs as datasets (the reference's ``gen`` plants Walsh amplitudes with
numpy noise and stays out of scope, as do snr / perf / iobench / coverage).
"""

from __future__ import annotations

import argparse
import json
import sys

import numpy as np

from . import dataset
from .errors import BadArguments, BigWHTError

JSON_SCHEMA_VERSION = 1


class _Usage(Exception):
    pass


class _Mismatch(Exception):
    """oracle --expect found a difference (exit 3, cli.py:255-257)."""


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise _Usage(message)


def _emit(args, command: str, payload: dict) -> None:
    if args.json:
        doc = {"schema_version": JSON_SCHEMA_VERSION, "command": command}
        doc.update(payload)
        print(json.dumps(doc, indent=2, sort_keys=True))


def _say(args, msg: str) -> None:
    if not args.quiet:
        print(msg, file=sys.stderr)


def _adopt_if_forced(args, path: str, assumed_domain: str) -> None:
    """cli.py:72-78: infer metadata for a bare payload only with --force."""
    import os

    if os.path.exists(dataset.sidecar_path(path)) or not args.force:
        return
    n = dataset.adopt(path, "int64", assumed_domain)
    _say(args, f"adopted bare payload {path}: assuming n={n}, int64, {assumed_domain} domain")


def cmd_transform_mem(args) -> None:
    """cli.py:144-172: load, transform on the GPU (bound checked), write back."""
    import torch

    from .core import Domain, Signal, _need_cuda, fwht_inplace
    from .parallel import log2_workers_for, plan_parallel, run_parallel

    _adopt_if_forced(args, args.in_path, "time")
    p = log2_workers_for(args.threads) if args.threads != 1 else 0
    arr, meta = dataset.open_memmap(args.in_path, "r+")
    if meta["domain"] != "time":
        raise BadArguments(f"{args.in_path} is already in the {meta['domain']} domain")
    _need_cuda()
    t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
    sig = Signal(t, Domain.TIME)
    if p == 0:
        fwht_inplace(sig)
    else:  # cli.py:157-160: the run_parallel schedule, here over 2**p shards on the GPU
        run_parallel(sig, plan_parallel(sig.log2_dim, p))
    arr[:] = sig.data.cpu().numpy()
    arr.flush()
    dataset.set_domain(args.in_path, "walsh")
    _emit(args, "transform mem", {"in": args.in_path, "n": meta["log2_dim"], "threads": args.threads,
                                  "device": torch.cuda.get_device_name()})
    _say(args, f"transformed {args.in_path} in GPU memory (threads={args.threads})")


def _refuse_interrupted(path: str, meta: dict, resume: bool) -> None:
    """A sidecar carrying the reference executor's pass-progress marker
    belongs to an interrupted out-of-core run: its payload is partially
    transformed although the domain still says time.  Refuse it with the
    reference's messages (external.py:155-178) instead of transforming it
    again; this engine cannot resume the reference's passes."""
    marker = meta.get("pass_progress")
    if marker is None:
        return
    if not resume:
        raise BadArguments(
            f"{path} has an interrupted transform "
            f"({marker.get('passes_done')}/{marker.get('total_passes')} "
            f"passes done); pass resume=True to continue")
    if marker.get("writing"):
        raise BadArguments(
            f"{path}: pass {marker.get('passes_done')} was interrupted "
            f"after its writes began, so the payload may be partially "
            f"transformed; re-running it would corrupt the data. Rebuild "
            f"the dataset from its source.")
    raise BadArguments(f"{path} has an interrupted transform of the reference's disk executor; "
                       "this engine keeps no pass-progress markers and cannot resume it")


def cmd_transform_ext(args) -> None:
    """cli.py:175-219: out-of-core through a device workspace of 2**B
    elements, streaming the memory-mapped payload (no resume markers)."""
    from .outofcore import fwht_out_of_core

    _adopt_if_forced(args, args.in_path, "time")
    _refuse_interrupted(args.in_path, dataset.read_meta(args.in_path), args.resume)
    if args.resume:
        raise BadArguments("--resume: this engine keeps no pass-progress markers (a run is one call)")
    if args.io_block_bytes is not None and (args.io_block_bytes < 8 or args.io_block_bytes % 8):
        raise BadArguments("--io-block-bytes must be a multiple of 8")
    if args.mem_log2 < 1:
        raise BadArguments(f"mem_log2 must be >= 1, got {args.mem_log2}")
    arr, meta = dataset.open_memmap(args.in_path, "r+")
    if meta["element_kind"] != "int64":
        raise BadArguments("the out-of-core transform is implemented for int64 datasets")
    if meta["domain"] != "time":
        raise BadArguments(f"{args.in_path} is already in the {meta['domain']} domain")
    # --mode entrywise|blocked and --io-block-bytes select the reference's
    # host I/O pattern; both run the same device passes here, which stream
    # the mapped payload in whole rows (every host pass moves each byte once).
    passes = fwht_out_of_core(arr, max(args.mem_log2, 15))
    arr.flush()
    dataset.set_domain(args.in_path, "walsh")
    _emit(args, "transform ext", {"in": args.in_path, "n": meta["log2_dim"], "mem_log2": args.mem_log2,
                                  "mode": args.mode, "passes": passes, "passes_executed": passes,
                                  "resumed_from": 0})
    _say(args, f"transformed {args.in_path} out of core: q={passes} passes ({passes} executed this run)")


def cmd_extract(args) -> None:
    """cli.py:260-291: |y| >= threshold, sorted by (-|y|, index), CSV or JSON.
    The payload is streamed through the GPU in blocks of 2**--block-log2."""
    import math

    import torch

    from .extract import extract_ge

    _adopt_if_forced(args, args.in_path, "walsh")
    arr, meta = dataset.open_memmap(args.in_path, "r")
    if meta["domain"] != "walsh":
        raise BadArguments(f"{args.in_path} is not Walsh-domain")
    if args.threshold < 0:
        raise BadArguments(f"tau must be >= 0, got {args.threshold}")
    # int64: |y| >= t  <=>  |y| >= ceil(t); float64 compares in double (noisy.py:218)
    tau = math.ceil(args.threshold) if meta["element_kind"] == "int64" else float(args.threshold)
    n = meta["log2_dim"]
    block = 1 << min(n, args.block_log2)
    hits = []
    for start in range(0, 1 << n, block):
        t = torch.from_numpy(np.array(arr[start:start + block])).cuda()
        i, v = extract_ge(t, tau, base=start)
        hits += list(zip(i.tolist(), v.tolist()))
    hits.sort(key=lambda h: (-abs(h[1]), h[0]))
    if args.json:
        _emit(args, "extract", {"in": args.in_path, "threshold": args.threshold, "count": len(hits),
                                "coefficients": [{"index": i, "coefficient": v} for i, v in hits]})
        return
    text = "index,coefficient\n" + "".join(f"{i},{v}\n" for i, v in hits)
    if args.out:
        with open(args.out, "w", encoding="utf-8") as f:
            f.write(text)
        _say(args, f"wrote {len(hits)} coefficients to {args.out}")
    else:
        sys.stdout.write(text)


def cmd_oracle(args) -> None:
    """cli.py:225-257: brute-force transform (O(4**n), on the GPU) written
    to --out and/or compared with --expect (exit 3 on a mismatch)."""
    from .core import Domain, Signal, wht_bruteforce

    if args.out_path is None and args.expect_path is None:
        raise _Usage("need --out and/or --expect")
    _adopt_if_forced(args, args.in_path, "time")
    arr, kind, domain = dataset.read_signal(args.in_path)
    result = wht_bruteforce(Signal(arr, Domain.TIME), limit=args.limit)
    matches = None
    if args.expect_path is not None:
        other, _, _ = dataset.read_signal(args.expect_path)
        matches = bool(np.array_equal(result.data, other))
    if args.out_path is not None:
        dataset.write_signal(args.out_path, result.data, domain="walsh")
    _emit(args, "oracle", {"in": args.in_path, "out": args.out_path, "expect": args.expect_path,
                           "matches": matches})
    if not args.json and matches is not None:
        print("match" if matches else "MISMATCH")
    if matches is False:
        raise _Mismatch()


def cmd_fold(args) -> None:
    """cli.py:477-518: fold a time-domain dataset through a GF(2) map
    (x'[L.j] += x[j], subspace.py:150-184) on the GPU."""
    import os

    import torch

    from . import subspace
    from .core import Domain, Signal

    _adopt_if_forced(args, args.in_path, "time")
    arr, meta = dataset.open_memmap(args.in_path, "r")
    if meta["domain"] != "time":
        raise BadArguments(f"{args.in_path} is not time-domain")
    if args.gen_dout is not None:
        if os.path.exists(args.matrix_path):
            raise BadArguments(f"--gen-dout refuses to overwrite {args.matrix_path}")
        rows = subspace.random_full_rank(meta["log2_dim"], args.gen_dout,
                                         args.seed if args.fold_seed is None else args.fold_seed)
        subspace.save_map(rows, args.matrix_path)
    else:
        rows = subspace.load_map(args.matrix_path)
    x = torch.from_numpy(np.array(arr)).cuda()  # read-only map: copy before handing to torch
    folded = subspace.fold(Signal(x, Domain.TIME), rows).data.cpu().numpy()
    dataset.write_signal(args.out_path, folded, domain="time")
    _emit(args, "fold", {"in": args.in_path, "matrix": args.matrix_path, "out": args.out_path,
                         "d_in": int(rows.shape[1]), "d_out": int(rows.shape[0])})
    _say(args, f"folded {args.in_path} ({rows.shape[1]} -> {rows.shape[0]} bits) into {args.out_path}")


def cmd_gen_config(args) -> None:
    """Write BASELINE.json config ``--config`` (optionally at size --n) as a
    time-domain int64 dataset, generated on the GPU."""
    from . import signals

    spec = signals.config(args.config, args.n)
    x = signals.make(spec).cpu().numpy()
    dataset.write_signal(args.out, x, domain="time")
    _emit(args, "gen-config", {"config": args.config, "n": spec.n, "out": args.out,
                               "planted": spec.masks, "threshold": spec.threshold})
    _say(args, f"wrote {args.out}: config {args.config}, n={spec.n}")


def build_parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="paper_1607_01039_b200", description="Exact Walsh-Hadamard transforms on B200.")
    ap.add_argument("--quiet", action="store_true", help="Suppress progress diagnostics.")
    ap.add_argument("--json", action="store_true", help="Emit machine-readable JSON.")
    ap.add_argument("--seed", type=int, default=0, help="Default seed for subcommands that use randomness.")
    ap.add_argument("--force", action="store_true",
                    help="Adopt bare payloads missing a sidecar, inferring n from the file size (int64).")
    sub = ap.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    tr = sub.add_parser("transform", help="Transform a dataset in place (time -> Walsh).")
    trs = tr.add_subparsers(dest="mode", required=True, parser_class=_Parser)
    m = trs.add_parser("mem", help="Whole dataset in GPU memory.")
    m.add_argument("--in", dest="in_path", required=True)
    m.add_argument("--threads", type=int, default=1, help="Workers of the run_parallel schedule (power of two).")
    m.set_defaults(func=cmd_transform_mem)
    e = trs.add_parser("ext", help="Out of core through a 2**B-element device workspace.")
    e.add_argument("--in", dest="in_path", required=True)
    e.add_argument("--mem-log2", "-b", dest="mem_log2", type=int, required=True)
    e.add_argument("--mode", choices=["entrywise", "blocked"], default="blocked")
    e.add_argument("--io-block-bytes", dest="io_block_bytes", type=int, default=None)
    e.add_argument("--resume", action="store_true")
    e.set_defaults(func=cmd_transform_ext)
    o = sub.add_parser("oracle", help="Brute-force reference transform (O(4**n); verification only).")
    o.add_argument("--in", dest="in_path", required=True)
    o.add_argument("--out", dest="out_path", default=None)
    o.add_argument("--expect", dest="expect_path", default=None)
    o.add_argument("--limit", type=int, default=14)
    o.set_defaults(func=cmd_oracle)
    f = sub.add_parser("fold", help="Fold a signal through a GF(2) linear reduction.")
    f.add_argument("--in", dest="in_path", required=True)
    f.add_argument("--matrix", dest="matrix_path", required=True)
    f.add_argument("--out", dest="out_path", required=True)
    f.add_argument("--gen-dout", dest="gen_dout", type=int, default=None)
    f.add_argument("--seed", dest="fold_seed", type=int, default=None)
    f.set_defaults(func=cmd_fold)
    x = sub.add_parser("extract", help="Walsh coefficients with |y| >= threshold as CSV.")
    x.add_argument("--in", dest="in_path", required=True)
    x.add_argument("--threshold", type=float, required=True)
    x.add_argument("--out", default=None)
    x.add_argument("--block-log2", type=int, default=28)
    x.set_defaults(func=cmd_extract)
    g = sub.add_parser("gen-config", help="Write a BASELINE.json config signal as a dataset.")
    g.add_argument("--config", type=int, required=True, choices=[1, 2, 3, 4, 5])
    g.add_argument("--n", type=int, default=None)
    g.add_argument("--out", required=True)
    g.set_defaults(func=cmd_gen_config)
    return ap


def run(argv=None) -> int:
    """Returns the exit code instead of raising SystemExit (cli.py:561-584)."""
    try:
        args = build_parser().parse_args(argv)
    except _Usage as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return 1
    try:
        args.func(args)
        return 0
    except _Usage as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return 1
    except _Mismatch:
        return 3
    except BigWHTError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return exc.exit_code
    except OSError as exc:
        print(f"I/O error: {exc}", file=sys.stderr)
        return 2


def main() -> None:
    sys.exit(run())
