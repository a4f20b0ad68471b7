"""Instruction-class histogram of the shipped pass kernels' SASS
(cuobjdump -sass of lib/libbigwht_b200.so), for the kernels of the n = 32
and n = 34 default plans.  It documents what the hot loops are made of:
LDG/STG (8- or 16-byte global accesses), STS/LDS (shared-memory transposes),
the DSMEM exchange (STAS = st.async to a partner CTA's shared memory,
SYNCS = the mbarrier arrive / try_wait, UCGABAR = the cluster barrier),
IADD3/IADD.64 (the butterflies), and the absence of UTMALDG / UBLKCP (TMA)
and of tcgen05 (UTCMMA): the passes are HBM-bound integer add/sub and keep
plain LDG/STG by measurement.

    python tools/sass_histogram.py [--lib path] [--out profiles/r02_sass_histogram.md]
"""
import argparse
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# mangled-name fragments of the kernels in the default plans (bw_abi.cu)
KERNELS = [
    ("k_pass<CfgLow13, 13> (n = 32 pass 1, low 13 bits)", r"k_passINS_8CfgLow13ELi13ELb0ELi0ELb0E"),
    ("k_pass<CfgLow14c, 14> (n = 34 pass 1, low 14 bits, 2-CTA)", r"k_passINS_9CfgLow14cELi14ELb0ELi0ELb0E"),
    ("k_pass_split<CfgHigh14cS, 4, A = 5> (n = 32/33 pass 2: split r = 10, 2-CTA)",
     r"k_pass_splitINS_11CfgHigh14cSELi4ELb0ELi5E"),
    ("k_pass_split<CfgHigh14cS, 4, A = 4> (n = 34 pass 2: split r = 10, 2-CTA)",
     r"k_pass_splitINS_11CfgHigh14cSELi4ELb0ELi4E"),
    ("k_pass_split<CfgHigh14cS, 4> offset table (round 1's split kernel, fallback)",
     r"k_pass_splitINS_11CfgHigh14cSELi4ELb0ELi0E"),
    ("k_pass<CfgHigh14c, 5> (n = 32 pass 3, r = 9, 2-CTA)", r"k_passINS_10CfgHigh14cELi5ELb0ELi0ELb0E"),
    ("k_pass<CfgHigh14c, 4> (n = 33/34 pass 3, r = 10, 2-CTA)", r"k_passINS_10CfgHigh14cELi4ELb0ELi0ELb0E"),
    # the compact plan's int32 engine (bw_kernels32.cuh; the default at n = 26..34 on small-valued signals)
    ("k32_first<5, CHECK> (compact pass 1 at n = 31..34: int64 -> int32, 9 rows, input test)", r"k32_firstILi5ELi1ELi4E"),
    ("k32_first<5, PLAIN> (the same, known bound)", r"k32_firstILi5ELi0ELi4E"),
    ("k32_first<6, CHECK> (compact pass 1 at n = 28..30: 8 rows)", r"k32_firstILi6ELi1ELi4E"),
    ("k32_high<5> (compact pass 2 at n = 32: int32 -> int32, 9 rows)", r"k32_highILi5ELi2E"),
    ("k32_high<6> (compact pass 2 at n = 30, 31, 33, 34: 8 rows)", r"k32_highILi6ELi2E"),
    ("k32_reg<3> (compact pass 3 at n = 34: 3 rows in registers)", r"k32_regILi3E"),
    ("k32_low (compact last pass: int32 -> int64, low 14 bits)", r"k32_lowILb0E"),
    ("k32_low<EX> (the same with the fused threshold extraction)", r"k32_lowILb1E"),
]

GROUPS = [
    ("LDG (global load)", r"^LDG\."),
    ("STG (global store)", r"^STG"),
    ("LDS (shared load)", r"^LDS"),
    ("STS (shared store)", r"^STS"),
    ("LDGSTS (cp.async global -> shared)", r"^LDGSTS"),
    ("STAS (st.async to a cluster partner)", r"^STAS"),
    ("SYNCS (mbarrier)", r"^SYNCS"),
    ("UCGABAR (cluster barrier)", r"^UCGABAR"),
    ("BAR (CTA barrier)", r"^BAR"),
    ("IADD3 / IADD / IMAD.IADD (butterfly add/sub)", r"^(IADD|IMAD\.IADD)"),
    ("VIMNMX3 (3-input max: the input test)", r"^VIMNMX3"),
    ("UTMALDG / UTMASTG / UBLKCP (TMA)", r"^(UTMA|UBLKCP)"),
    ("UTC* (tcgen05)", r"^UTC"),
]


def functions(sass: str):
    cur, body = None, []
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if cur and m:
            body.append(m.group(2))
    if cur:
        yield cur, body


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_1607_01039_b200", "lib", "libbigwht_b200.so"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sass_histogram.md"))
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.lib], check=True, capture_output=True, text=True).stdout
    funcs = dict(functions(sass))
    lines = ["# SASS instruction histogram of the default-plan pass kernels (sm_100a)", "",
             f"`cuobjdump -sass {os.path.relpath(a.lib, ROOT)}` (tools/sass_histogram.py). Static counts per "
             "kernel body (fully unrolled: one tile per CTA).", ""]
    hdr = "| kernel | registers | total | " + " | ".join(g for g, _ in GROUPS) + " | widest LDG / STG |"
    lines += [hdr, "|" + "---|" * (len(GROUPS) + 4)]
    res = subprocess.run(["cuobjdump", "-res-usage", a.lib], capture_output=True, text=True).stdout
    regs = dict(re.findall(r"Function (\S+):\s+REG:(\d+)", res))
    for title, pat in KERNELS:
        name = next((f for f in funcs if re.search(pat, f)), None)
        if name is None:
            lines.append(f"| {title} | (not found) |" + " |" * (len(GROUPS) + 2))
            continue
        ops = funcs[name]
        cnt = collections.Counter()
        for op in ops:
            for g, rx in GROUPS:
                if re.match(rx, op):
                    cnt[g] += 1
        ldg = sorted({op for op in ops if op.startswith("LDG.")})
        stg = sorted({op for op in ops if op.startswith("STG")})
        lines.append(f"| {title} | {regs.get(name, '?')} | {len(ops)} | " + " | ".join(str(cnt[g]) for g, _ in GROUPS)
                     + f" | {', '.join(ldg)} / {', '.join(stg)} |")
    lines += ["", "Reading: every tile element is loaded and stored once (32 LDG.E.64 or 16 LDG.E.128 per "
              "thread); the 2-CTA kernels move half the tile through DSMEM with STAS and wait on one "
              "mbarrier (SYNCS) after a split cluster barrier (UCGABAR arrive / wait). No TMA or tcgen05 "
              "instruction appears: `tools/mb_tma.cu` / `mb_bulk.cu` measured TMA tiles and bulk copies "
              "below plain LDG/STG for these row shapes (profiles/r01_mb_tma.log, r01_mb_bulk.log), and "
              "the transform has nothing to multiply.", "",
              "The int32 engine's kernels (k32_*, one CTA per 2^14-element tile, no cluster): k32_first stages "
              "half of its int64 tile through shared memory with 16 LDGSTS (cp.async, 16 bytes each) next to 16 "
              "LDG.128, so the checked pass keeps the whole tile in flight; its input test is a 64-bit add plus "
              "LOP3 / VIMNMX3 per pair of values; the int32 butterflies are IADD3 / IMAD.IADD on 32-bit "
              "registers; k32_reg has no shared-memory instruction at all."]
    with open(a.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
