"""Command line on the GPU engine: ``python -m paper_1607_01039_b200 ...``.

Mirrors the reference CLI's transform / extract commands
(/root/reference/pkg/src/bigwht/cli.py:144-291) on the reference's dataset
format: the same options, exit codes (0 ok, 1 usage, 2 I/O, 3 validation;
cli.py:561-584), stderr diagnostics suppressed by --quiet and the
``--json`` schema-version-1 documents.  ``gen-config`` writes the seeded
BASELINE.json configs as datasets (the reference's ``gen`` plants Walsh
amplitudes with numpy noise and stays out of scope).
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


def cmd_transform_mem(args) -> None:
    """cli.py:144-172: load, transform on the GPU (bound checked), write back."""
    import torch

    from .core import Domain, Signal, fwht_inplace

    arr, meta = dataset.open_memmap(args.in_path, "r+")
    if meta["domain"] != "time":
        raise BadArguments(f"{args.in_path} is already in the {meta['domain']} domain")
    t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
    sig = fwht_inplace(Signal(t, Domain.TIME))
    arr[:] = sig.data.cpu().numpy()
    arr.flush()
    dataset.set_domain(args.in_path, "walsh")
    _emit(args, "transform mem", {"in": args.in_path, "n": meta["log2_dim"], "device": torch.cuda.get_device_name()})
    _say(args, f"transformed {args.in_path} in GPU memory")


def cmd_transform_ext(args) -> None:
    """cli.py:175-219: out-of-core through a device workspace of 2**B
    elements, streaming the memory-mapped payload (no resume markers)."""
    from .outofcore import fwht_out_of_core

    arr, meta = dataset.open_memmap(args.in_path, "r+")
    if meta["element_kind"] != "int64":
        raise BadArguments("the out-of-core transform is implemented for int64 datasets")
    if meta["domain"] != "time":
        raise BadArguments(f"{args.in_path} is already in the {meta['domain']} domain")
    passes = fwht_out_of_core(arr, args.mem_log2)
    arr.flush()
    dataset.set_domain(args.in_path, "walsh")
    _emit(args, "transform ext", {"in": args.in_path, "n": meta["log2_dim"], "mem_log2": args.mem_log2,
                                  "passes": passes})
    _say(args, f"transformed {args.in_path} out of core: {passes} passes")


def cmd_extract(args) -> None:
    """cli.py:260-291: |y| >= threshold, sorted by (-|y|, index), CSV or JSON.
    The payload is streamed through the GPU in blocks of 2**--block-log2."""
    import math

    import torch

    from .extract import extract_ge

    arr, meta = dataset.open_memmap(args.in_path, "r")
    if meta["domain"] != "walsh":
        raise BadArguments(f"{args.in_path} is not Walsh-domain")
    if meta["element_kind"] != "int64":
        raise BadArguments("GPU extraction is implemented for int64 datasets")
    if args.threshold < 0:
        raise BadArguments(f"tau must be >= 0, got {args.threshold}")
    tau = math.ceil(args.threshold)
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
    sub = ap.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    tr = sub.add_parser("transform", help="Transform a dataset in place (time -> Walsh).")
    trs = tr.add_subparsers(dest="mode", required=True, parser_class=_Parser)
    m = trs.add_parser("mem", help="Whole dataset in GPU memory.")
    m.add_argument("--in", dest="in_path", required=True)
    m.set_defaults(func=cmd_transform_mem)
    e = trs.add_parser("ext", help="Out of core through a 2**B-element device workspace.")
    e.add_argument("--in", dest="in_path", required=True)
    e.add_argument("--mem-log2", "-b", dest="mem_log2", type=int, required=True)
    e.set_defaults(func=cmd_transform_ext)
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
    except BigWHTError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return exc.exit_code
    except OSError as exc:
        print(f"I/O error: {exc}", file=sys.stderr)
        return 2


def main() -> None:
    sys.exit(run())
