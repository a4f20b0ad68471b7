"""One small invocation of each kernel family, checked against the oracle --
the target of the compute-sanitizer runs (tools/gpu_sanitize.sh):

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py --family split

Families (the kernel templates of csrc/bw_kernels.cuh they launch):
  low1      k_pass<CfgLow13> + k_pass<CfgHigh13> + k_pass<CfgReg>   (1-CTA tiles)
  cluster   k_pass<CfgLow14c> + k_pass<CfgHigh14c> (2-CTA DSMEM st.async / mbarrier),
            k_pass<CfgLow15c> + k_pass<CfgHigh15c> (4-CTA)
  split     k_pass_split<CfgHigh13S / CfgHigh14cS>
  split_ct  k_pass_split<CfgHigh14cS, L, EX, A> (compile-time low run, the n = 32..34 plans)
  compact   k_pass_map<..., MAP_CHECK / MAP_RESTORE> + the compact plan's passes
  bound     k_pass<low, MAP_CHECK / MAP_RESTORE> (fwht_inplace's fused bound check)
  two_pass  k_two_pass (cooperative grid sync)
  map       k_pass_map<..., TPC=2> (narrow intermediates: per-tile mbarrier phase re-arm on clusters)
  xfused    k_pass_x (fused cross-shard pass, P = 2 / 4 shards on one device) + extraction epilogue
  narrow    k_pack_narrow + k_xshard_narrow + widening k_pass<..., SB = 1>
  extract   k_pass<..., EX = true> + k_sort_hits, k_extract_count / scan / write
  fold      k_fold_blocks, k_fold<smem bins>
  aux       k_minmax, k_small, k_bruteforce, k_sumsq, float64 passes, inverse
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1607_01039_b200 as bw  # noqa: E402
from oracle import load_c, oracle_np  # noqa: E402
from paper_1607_01039_b200 import _lib, sharded, subspace  # noqa: E402

C = load_c()
SH = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731


def ref_fwht(x):
    y = x.copy()
    C.oracle_fwht_i64(y.ctypes.data, int(y.size).bit_length() - 1)
    return y


def planned(x, plan):
    t = torch.from_numpy(x.copy()).cuda()
    n = int(t.numel()).bit_length() - 1
    arr = (ctypes.c_int * len(plan))(*plan)
    _lib.check(_lib.lib().bw_fwht_i64_planned(t.data_ptr(), n, arr, len(plan), SH()))
    return t.cpu().numpy()


def check(name, ok):
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        raise SystemExit(1)


def split(r, q, a, k2):
    return r | ((q + 1) << 4) | (a << 8) | (k2 << 12)


def fam_low1():
    n = 20
    x = oracle_np.gen(2, 1, [1 << 20], 0, 1 << n)
    ref = ref_fwht(x)
    check("low13 + high r=7 (1 CTA)", np.array_equal(planned(x, [13, 7 | (1 << 4)]), ref))
    check("low13 + reg r=3 + reg r=4", np.array_equal(planned(x, [13, 3, 4]), ref))


def fam_cluster():
    n = 24
    x = oracle_np.gen(2, 2, [1 << 20], 0, 1 << n)
    ref = ref_fwht(x)
    check("low14 (2-CTA) + high r=10 (2-CTA)", np.array_equal(planned(x, [14, 10 | (2 << 4)]), ref))
    check("low13 + high r=9 (2-CTA) + 2", np.array_equal(planned(x, [13, 9 | (2 << 4), 2]), ref))
    check("low15 (4-CTA) + high r=9 (4-CTA)", np.array_equal(planned(x, [15, 9 | (3 << 4)]), ref))


def fam_split():
    n = 24
    x = oracle_np.gen(2, 3, [1 << 20], 0, 1 << n)
    ref = ref_fwht(x)
    check("split r=9 on 2 CTAs", np.array_equal(planned(x, [13, split(9, 1, 4, 19), 2]), ref))
    check("split r=6 on 1 CTA", np.array_equal(planned(x, [13, split(6, 0, 3, 21), 5]), ref))


def fam_split_ct():
    """k_pass_split with a compile-time low run (A = 1..9 on 10 rows, 1..8 on 9)."""
    n = 26
    x = oracle_np.gen(2, 12, [1 << 20], 0, 1 << n)
    ref = ref_fwht(x)
    for a in (1, 4, 5, 9):
        check(f"split r=10 a={a} (compile-time offsets)",
              np.array_equal(planned(x, [13, split(10, 1, a, 26 - (10 - a)), 3]), ref))
    check("split r=9 a=4", np.array_equal(planned(x, [13, split(9, 1, 4, 21), 4]), ref))


def fam_compact():
    """The compact in-place plan: checked first pass (cluster agreement through
    DSMEM flags), the exact restore after an abort, unchecked passes."""
    n = 24
    lim = int(_lib.lib().bw_compact_limit(n))
    x = oracle_np.gen(2, 13, [lim], 0, 1 << n)
    for bound in (-1, lim):
        t = torch.from_numpy(x.copy()).cuda()
        bw.fwht_array(t, compact=True if bound < 0 else bound)
        check(f"compact plan (bound {bound}) used={bw.core.last_compact}",
              bw.core.last_compact and np.array_equal(t.cpu().numpy(), ref_fwht(x)))
    y = x.copy()
    y[(1 << n) - 5] = lim + 1  # the last tiles abort: most tiles are written, then restored
    t = torch.from_numpy(y.copy()).cuda()
    bw.fwht_array(t, compact=True)
    check("compact fallback (restore + int64 plan)",
          not bw.core.last_compact and np.array_equal(t.cpu().numpy(), ref_fwht(y)))
    # the int32 engine's first pass (k32_first<6> / <5>: half of the tile landing in shared memory
    # through cp.async, the verdict on the inter-round barrier), k32_restore, k32_high, k32_low
    for n in (22, 23, 26):
        lim = int(_lib.lib().bw_compact_limit(n))
        x = oracle_np.gen(2, 17 + n, [min(lim, 1 << 20)], 0, 1 << n)
        ref = ref_fwht(x)
        for bound in (-1, lim):
            t = torch.from_numpy(x.copy()).cuda()
            bw.fwht_array(t, compact=True if bound < 0 else bound)
            check(f"int32-engine compact plan n={n} (bound {bound})",
                  bw.core.last_compact and np.array_equal(t.cpu().numpy(), ref))
        y = x.copy()
        y[(1 << n) - 5] = lim + 1
        t = torch.from_numpy(y.copy()).cuda()
        bw.fwht_array(t, compact=True)
        check(f"int32-engine compact fallback n={n} (k32_restore + int64 plan)",
              not bw.core.last_compact and np.array_equal(t.cpu().numpy(), ref_fwht(y)))
    n = 26  # the threshold extraction in k32_low's final registers (the default at this size)
    x = oracle_np.gen(1, 3, [], 0, 1 << n)
    x[::4099] = 1
    ref = ref_fwht(x)
    tau = int(np.sort(np.abs(ref))[-40])
    t = torch.from_numpy(x.copy()).cuda()
    i, v = bw.fwht_extract_ge(t, tau)
    hits = np.nonzero(np.abs(ref) >= tau)[0]
    check("fused extraction in k32_low", np.array_equal(t.cpu().numpy(), ref) and i.cpu().tolist() == hits.tolist()
          and v.cpu().tolist() == ref[hits].tolist())


def fam_bound():
    """fwht_inplace's low pass with the bound fused in (k_pass<..., MAP_CHECK>
    and the MAP_RESTORE pass after a violation), 1- and 2-CTA low passes."""
    for n in (22, 24):
        edge = (1 << (63 - n)) - 1
        x = oracle_np.gen(2, 14 + n, [1 << 20], 0, 1 << n)
        s = bw.fwht_inplace(bw.Signal(torch.from_numpy(x.copy()).cuda()))
        check(f"fused bound n={n}", np.array_equal(s.data.cpu().numpy(), ref_fwht(x)))
        y = x.copy()
        y[(1 << n) - 9] = edge + 1
        t = torch.from_numpy(y.copy()).cuda()
        try:
            bw.fwht_inplace(bw.Signal(t))
            ok = False
        except bw.errors.OverflowBoundError:
            ok = np.array_equal(t.cpu().numpy(), y)
        check(f"fused bound violation restored n={n}", ok)


def fam_two_pass():
    for n in (16, 18, 20):
        x = oracle_np.gen(2, 4, [1 << 20], 0, 1 << n)
        t = torch.from_numpy(x.copy()).cuda()
        bw.fwht_array(t)  # n = 16..20: both passes in one cooperative launch
        check(f"k_two_pass n={n}", np.array_equal(t.cpu().numpy(), ref_fwht(x)))


def fam_map():
    n = 22
    x = oracle_np.gen(1, 5, [], 0, 1 << n)
    t = torch.from_numpy(x.copy()).cuda()
    bw.fwht_array(t, narrow=True)
    check(f"narrow intermediates (TPC={os.environ.get('BW_NARROW_TPC', '2')}) used={bw.core.last_narrow}",
          np.array_equal(t.cpu().numpy(), ref_fwht(x)) and bw.core.last_narrow)


def fam_xfused():
    n = 22
    x = oracle_np.gen(2, 6, [1 << 20], 0, 1 << n)
    ref = ref_fwht(x)
    for p in (1, 2):
        shards = [torch.from_numpy(c.copy()).cuda() for c in np.split(x, 1 << p)]
        sharded.fwht_shards(shards, fused=True)
        check(f"k_pass_x P={1 << p}", np.array_equal(np.concatenate([s.cpu().numpy() for s in shards]), ref))
    tau = 5_000_000_000  # ~4 sigma of the uniform(+-2^20) signal's coefficients
    shards = [torch.from_numpy(c.copy()).cuda() for c in np.split(x, 2)]
    i, v = sharded.fwht_shards_extract_ge(shards, tau)
    wi, wv = oracle_np.extract_gt_by_index(ref, tau - 1)
    check("k_pass_x extraction epilogue", i.cpu().tolist() == wi.tolist() and v.cpu().tolist() == wv.tolist())


def fam_narrow():
    n = 22
    x = oracle_np.gen(1, 7, [], 0, 1 << n)
    shards = [torch.from_numpy(c.copy()).cuda() for c in np.split(x, 4)]
    sharded.fwht_shards(shards, narrow=True)
    check("narrow wire P=4", np.array_equal(np.concatenate([s.cpu().numpy() for s in shards]), ref_fwht(x)))


def fam_extract():
    n = 22
    x = oracle_np.gen(2, 8, [1 << 10], 0, 1 << n)
    ref = ref_fwht(x)
    tau = 1 << 22
    t = torch.from_numpy(x.copy()).cuda()
    i, v = bw.fwht_extract_ge(t, tau)
    wi, wv = oracle_np.extract_gt_by_index(ref, tau - 1)
    check("fused extraction", i.cpu().tolist() == wi.tolist() and v.cpu().tolist() == wv.tolist())
    i2, v2 = bw.extract_ge(t, tau)
    check("ordered extraction", i2.cpu().tolist() == wi.tolist())


def fam_fold():
    n = 22
    x = oracle_np.gen(2, 9, [1 << 10], 0, 1 << n)
    for d in (6, 10, 16):
        rows = oracle_np.random_full_rank(n, d, 3 + d)
        got = subspace.fold(bw.Signal(torch.from_numpy(x.copy()).cuda()), rows).data.cpu().numpy()
        check(f"fold d_out={d}", np.array_equal(got, oracle_np.fold(x, rows)))


def fam_aux():
    n = 14
    x = oracle_np.gen(2, 10, [1 << 20], 0, 1 << n)
    t = torch.from_numpy(x.copy()).cuda()
    bw.check_magnitude_bound(t, n)
    s = bw.fwht_inplace(bw.Signal(t))
    check("bound + transform", np.array_equal(s.data.cpu().numpy(), ref_fwht(x)))
    bw.inverse_wht_inplace(s)
    check("inverse", np.array_equal(s.data.cpu().numpy(), x))
    check("parseval", bw.parseval_energy(bw.Signal(torch.from_numpy(x.copy()).cuda())) == int((x.astype(object) ** 2).sum()))
    small = oracle_np.gen(2, 11, [100], 0, 1 << 8)
    check("bruteforce + k_small", np.array_equal(bw.wht_bruteforce(bw.Signal(small.copy())).data, ref_fwht(small)))
    f = np.random.default_rng(1).normal(size=1 << 20)
    g = torch.from_numpy(f.copy()).cuda()
    bw.fwht_array(g)
    fr = f.copy()
    C.oracle_fwht_f64(fr.ctypes.data, 20)
    check("float64 passes", np.array_equal(g.cpu().numpy().view(np.int64), fr.view(np.int64)))


FAMILIES = {k[4:]: v for k, v in globals().items() if k.startswith("fam_")}

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--family", default="all", choices=["all", *FAMILIES])
    a = ap.parse_args()
    for name, fn in FAMILIES.items():
        if a.family in ("all", name):
            fn()
    torch.cuda.synchronize()
    print("done", a.family)
