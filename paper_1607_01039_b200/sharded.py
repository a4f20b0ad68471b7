"""Multi-GPU FWHT: the top log2(P) index bits sharded over P devices.

Reference: the data-parallel schedule of
/root/reference/pkg/src/bigwht/parallel.py:87-111 with m = P workers.  Its
phase 0 (2**p independent chunk WHTs over the low n-p bits) is each GPU's
local transform; its p stage phases k = n-p .. n-1 are fused here into ONE
cross-shard P-point butterfly (kernel K6): every local index i is owned by
exactly one GPU g (slice g of the local index range), which gathers the P
values shards[r][i] over NVLink, butterflies them and scatters them back.
The slices are disjoint, which is the check_disjoint argument of
parallel.py:114-134, so the in-place exchange needs only two barriers
(before: every local transform done; after: every exchange done).

The exchange can also be FUSED into the last local pass (kernel K6',
``bw_fwht_xfused_pass_i64``): the last local high pass's tile is extended
with the P shard bits, so one kernel loads its rows from every shard over
NVLink, applies the last local stages and the log2 P cross stages, and
stores back -- one HBM round trip fewer than local passes + a separate
exchange.  ``fused=True`` / ``mode="fused"`` select it.

NARROW WIRE (``mode="narrow"``): the log2 P cross-shard stages run FIRST,
on the untransformed input (int64 stages on distinct bits commute, so the
result is still bit-identical).  When every |x| <= floor(127 / P) (a +-1
Boolean signal, the paper's use case), no intermediate of the P-point
butterfly leaves int8, so each shard is packed to one byte per point, the
exchange moves 1 byte per point over NVLink instead of 8, and every device
then transforms its shard locally, the first pass widening the packed
bytes (bw_fwht_widen).  Larger inputs fall back to the fused int64 path
(the pack kernel flags them; the shards are untouched).

Three drivers share these kernels:
  * ``fwht_shards``      -- one process, shards on one or several devices
                            (single-GPU P-shard emulation, or P2P over NVLink).
  * ``fwht_distributed`` -- one process per GPU (torch.distributed):
      mode="fused" (default): local passes, then K6' over peer pointers;
      mode="peer": CUDA IPC peer pointers, the K6 kernel reads and writes the
                   peers' HBM directly over NVLink (fused compute+exchange);
      mode="a2a":  all-to-all transpose + local K6 on the receive slots +
                   all-to-all back (NCCL on GPUs; gloo on CPU for tests);
      mode="narrow": the int8 exchange first, then the local transforms.
"""

from __future__ import annotations

import ctypes
import json

import torch

from . import _lib
from .core import _is_power_of_two, _stream_handle, fwht_array
from .errors import BadArguments, BigWHTError, DeviceError, InvalidWorkerCount


def log2_shards(p_count: int) -> int:
    """parallel.py:79-84 (log2_workers_for) with P = 1 allowed (no exchange)."""
    if p_count < 1 or not _is_power_of_two(p_count) or p_count > (1 << 3):
        raise InvalidWorkerCount(f"shard count must be a power of two in 1..8, got {p_count}")
    return p_count.bit_length() - 1


def plan(n: int, p: int) -> dict:
    """The device pass plan for a 2**n transform over 2**p shards
    (bw_plan_describe): local passes, cross-shard stages, bytes per pass."""
    buf = ctypes.create_string_buffer(4096)
    need = _lib.lib().bw_plan_describe(n, p, buf, len(buf))
    if need < 0:
        _lib.check(-need)
    return json.loads(buf.value.decode())


def plan_check(n: int, pass_bits=None) -> int:
    """Static checker of a local pass plan (bw_plan_check): every element
    touched once per pass, every stage exactly once; returns the butterfly
    count (= n * 2**(n-1), parallel.py:137-147 total_butterflies)."""
    bf = ctypes.c_uint64(0)
    if pass_bits:
        arr = (ctypes.c_int * len(pass_bits))(*pass_bits)
        _lib.check(_lib.lib().bw_plan_check(n, arr, len(pass_bits), ctypes.byref(bf)))
    else:
        _lib.check(_lib.lib().bw_plan_check(n, None, 0, ctypes.byref(bf)))
    return int(bf.value)


def slice_of(rank: int, world: int, local_len: int) -> tuple[int, int]:
    """[begin, begin+count) of the local index range owned by ``rank`` in the
    cross-shard stage (even-sized, disjoint, covering)."""
    pairs = local_len // 2
    lo = pairs * rank // world
    hi = pairs * (rank + 1) // world
    return 2 * lo, 2 * (hi - lo)


def fused_plan(n_local: int, p: int) -> tuple[list[int], int]:
    """(local pass widths, r_last) of the fused multi-device plan."""
    widths = (ctypes.c_int * 8)()
    nw = ctypes.c_int(8)
    r = ctypes.c_int(0)
    _lib.check(_lib.lib().bw_plan_fused(n_local, p, widths, ctypes.byref(nw), ctypes.byref(r)))
    return [widths[i] for i in range(nw.value)], int(r.value)


def plan_check_fused(n_local: int, p: int) -> int:
    """Static checker of the fused multi-device plan (bw_plan_check_fused)."""
    bf = ctypes.c_uint64(0)
    _lib.check(_lib.lib().bw_plan_check_fused(n_local, p, ctypes.byref(bf)))
    return int(bf.value)


def _local_partial(t: torch.Tensor, n_local: int, widths: list[int]) -> None:
    arr = (ctypes.c_int * len(widths))(*widths)
    with torch.cuda.device(t.device):
        _lib.check(_lib.lib().bw_fwht_i64_partial(t.data_ptr(), n_local, arr, len(widths), _stream_handle(t)))


WIRE_BYTES = 1  # narrow wire: int8 (|x| <= 127 >> log2 P)


def narrow_ok(local_len: int, p: int) -> bool:
    """The narrow exchange needs 16-point-aligned slices of every shard."""
    return p > 0 and local_len % (16 << p) == 0


def _pack(t: torch.Tensor, packed: torch.Tensor, flag: torch.Tensor, p: int) -> None:
    with torch.cuda.device(t.device):
        _lib.check(_lib.lib().bw_pack_narrow_i64(t.data_ptr(), t.numel(), WIRE_BYTES, p, packed.data_ptr(),
                                                 flag.data_ptr(), _stream_handle(t)))


def _xshard_narrow(ptrs: list[int], p: int, begin: int, count: int, dev: torch.device) -> None:
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().bw_xshard_narrow(arr, WIRE_BYTES, p, begin, count,
                                               torch.cuda.current_stream(dev).cuda_stream))


def _widen(packed: torch.Tensor, t: torch.Tensor) -> None:
    n_local = t.numel().bit_length() - 1
    with torch.cuda.device(t.device):
        _lib.check(_lib.lib().bw_fwht_widen(packed.data_ptr(), WIRE_BYTES, t.data_ptr(), n_local,
                                            _stream_handle(t), None))


def _fused_pass(ptrs: list[int], p: int, n_local: int, r: int, rank: int, dev: torch.device) -> None:
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().bw_fwht_xfused_pass_i64(arr, p, n_local, r, rank,
                                                      torch.cuda.current_stream(dev).cuda_stream))


def _fused_pass_extract(ptrs: list[int], p: int, n_local: int, r: int, rank: int, dev: torch.device, tau: int,
                        idx: torch.Tensor, val: torch.Tensor, count: torch.Tensor) -> None:
    """K6' with |W| >= tau tested on its final values (hits appended with
    global indices, unordered; count accumulated on the device)."""
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().bw_fwht_xfused_pass_extract_i64(
            arr, p, n_local, r, rank, int(tau), 0, idx.data_ptr(), val.data_ptr(), idx.numel(), count.data_ptr(),
            torch.cuda.current_stream(dev).cuda_stream))


def _enable_peers(devices: list[int]) -> None:
    """Peer access between every pair of the devices holding shards (no-op
    for shards on one device): the K6 / K6' / narrow kernels on device d
    load and store the other devices' shards, and the fused extraction
    appends its hits into device 0's buffers."""
    if len(devices) < 2:
        return
    for d in devices:
        with torch.cuda.device(d):
            for q in devices:
                _lib.check(_lib.lib().bw_enable_peer_access(q))


def _check_shards(shards: list[torch.Tensor]) -> int:
    local = shards[0].numel()
    for s in shards:
        if s.numel() != local or s.dtype != torch.int64 or not s.is_cuda or not s.is_contiguous():
            raise BadArguments("shards must be equal-length contiguous CUDA int64 tensors")
    return local


def fwht_shards_extract_ge(shards: list[torch.Tensor], tau: int, cap: int = 1 << 16):
    """fwht_shards(fused=True) with the extraction (|W| >= tau, noisy.py:185-222)
    fused into the cross-shard pass: returns (index, value) CUDA tensors of
    the whole 2**n signal, sorted by index."""
    p = log2_shards(len(shards))
    local = _check_shards(shards)
    n_local = local.bit_length() - 1
    if p == 0 or n_local < 14:
        raise BadArguments("fused extraction needs P >= 2 shards of >= 2**14 points")
    widths, r = fused_plan(n_local, p)
    for s in shards:
        _local_partial(s, n_local, widths)
    devices = sorted({s.device.index for s in shards})
    for d in devices:
        torch.cuda.synchronize(d)
    _enable_peers(devices)
    dev0 = shards[0].device
    idx = torch.empty(cap, dtype=torch.int64, device=dev0)
    val = torch.empty(cap, dtype=torch.int64, device=dev0)
    count = torch.zeros(1, dtype=torch.int64, device=dev0)
    ptrs = [s.data_ptr() for s in shards]
    for g, s in enumerate(shards):
        _fused_pass_extract(ptrs, p, n_local, r, g, s.device, tau, idx, val, count)
    for d in devices:
        torch.cuda.synchronize(d)
    k = int(count.item())
    if k > cap:
        raise BadArguments(f"{k} hits exceed the capacity {cap}")
    order = torch.argsort(idx[:k])
    return idx[:k][order], val[:k][order]


# ------------------------------------------------------- single process ---

def xshard(shards: list[torch.Tensor], begin: int = 0, count: int | None = None) -> None:
    """Kernel K6 over [begin, begin+count) of every shard, launched on the
    current device (all shard pointers must be accessible from it)."""
    p = log2_shards(len(shards))
    local = shards[0].numel()
    count = local - begin if count is None else count
    ptrs = (ctypes.c_void_p * len(shards))(*[s.data_ptr() for s in shards])
    dev = torch.cuda.current_device()
    _lib.check(_lib.lib().bw_xshard_i64(ptrs, p, begin, count,
                                        torch.cuda.current_stream(dev).cuda_stream))


def fwht_shards(shards: list[torch.Tensor], fused: bool = False, narrow: bool = False) -> int:
    """Transform the 2**n signal whose P = len(shards) contiguous shards are
    given (shard r = indices r*2**(n-p) ...), in place.  Shards may live on
    one device (emulation of P GPUs) or on P devices (P2P over NVLink).
    fused: K6' (last local pass + cross stages); narrow: the narrow-wire
    exchange first (falls back to fused when an input is too large).
    Returns n * 2**(n-1)."""
    p = log2_shards(len(shards))
    local = _check_shards(shards)
    n_local = local.bit_length() - 1
    devices = sorted({s.device.index for s in shards})
    if narrow and narrow_ok(local, p):
        packed = [torch.empty(local, dtype=torch.int8, device=s.device) for s in shards]
        flags = [torch.zeros(1, dtype=torch.int32, device=s.device) for s in shards]
        for s, pk, f in zip(shards, packed, flags):
            _pack(s, pk, f, p)
        if any(int(f.item()) for f in flags):  # (synchronises every device: barrier (i))
            return fwht_shards(shards, fused=True)
        _enable_peers(devices)
        ptrs = [pk.data_ptr() for pk in packed]
        m = local >> p
        for g, s in enumerate(shards):  # device g exchanges slice g of every packed shard
            _xshard_narrow(ptrs, p, g * m, m, s.device)
        for d in devices:  # barrier (ii)
            torch.cuda.synchronize(d)
        for s, pk in zip(shards, packed):
            _widen(pk, s)
        for d in devices:
            torch.cuda.synchronize(d)
        n = n_local + p
        return n << (n - 1)
    if fused and p > 0 and n_local >= 14:
        widths, r = fused_plan(n_local, p)
        for s in shards:  # local passes over the low n_local - r bits
            _local_partial(s, n_local, widths)
        for d in devices:
            torch.cuda.synchronize(d)
        _enable_peers(devices)
        ptrs = [s.data_ptr() for s in shards]
        for g, s in enumerate(shards):  # device g runs its share of K6'
            _fused_pass(ptrs, p, n_local, r, g, s.device)
        for d in devices:
            torch.cuda.synchronize(d)
        n = n_local + p
        return n << (n - 1)
    for s in shards:  # parallel.py phase 0: independent local transforms
        with torch.cuda.device(s.device):
            fwht_array(s)
    if p == 0:
        return (n_local) << max(n_local - 1, 0)
    if len(devices) > 1:
        for d in devices:  # barrier (i): every local transform done
            torch.cuda.synchronize(d)
        _enable_peers(devices)
    # Slice g of the local range is exchanged by the device of shard g.
    for g, s in enumerate(shards):
        b, c = slice_of(g, len(shards), local)
        with torch.cuda.device(s.device):
            xshard(shards, b, c)
    if len(devices) > 1:
        for d in devices:  # barrier (ii)
            torch.cuda.synchronize(d)
    n = n_local + p
    return n << (n - 1)


# -------------------------------------------------- one process per GPU ---

class CudaBackend:
    """Product compute backend: the sm_100a kernels through the C ABI."""

    def local_fwht(self, t: torch.Tensor) -> None:
        fwht_array(t)

    def xshard_slots(self, slots: torch.Tensor, p: int) -> None:
        """K6 over the P rows of a [P, m] receive buffer."""
        m = slots.shape[1]
        with torch.cuda.device(slots.device):
            _lib.check(_lib.lib().bw_xshard_strided_i64(slots.data_ptr(), m, p, 0, m,
                                                        _stream_handle(slots)))

    def sync(self, t: torch.Tensor) -> None:
        # the caller's stream only: copies of other signals on other streams
        # (fwht_distributed_many) keep running across the barriers
        torch.cuda.current_stream(t.device).synchronize()


class _PeerMap:
    """CUDA IPC mapping of every rank's shard into this process.  Collective:
    when any rank cannot export or map a shard (no IPC for the allocation, no
    peer access), every rank raises DeviceError, so callers can fall back
    together (bench.py drops to the NCCL all-to-all exchange)."""

    def __init__(self, local: torch.Tensor, group, dist):
        L = _lib.lib()
        handle = (ctypes.c_char * 64)()
        off = ctypes.c_uint64(0)
        try:
            _lib.check(L.bw_ipc_get_handle(local.data_ptr(), handle, ctypes.byref(off)))
            mine = (bytes(handle), int(off.value))
        except BigWHTError as e:
            mine = ("error", str(e))
        world = dist.get_world_size(group)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        bad = [r for r, h in enumerate(allh) if h[0] == "error"]
        if bad:
            raise DeviceError(f"CUDA IPC export failed on rank(s) {bad}: {allh[bad[0]][1]}")
        self.rank = dist.get_rank(group)
        self.ptrs, self.opened = [], []
        err = None
        for r, (h, o) in enumerate(allh):
            if r == self.rank:
                self.ptrs.append(local.data_ptr())
                continue
            ptr = ctypes.c_void_p(0)
            try:
                _lib.check(L.bw_ipc_open_handle(h, o, ctypes.byref(ptr)))
            except BigWHTError as e:
                err = str(e)
                break
            self.ptrs.append(ptr.value)
            self.opened.append((ptr.value, o))
        errs = [None] * world
        dist.all_gather_object(errs, err, group=group)
        if any(e is not None for e in errs):
            self.close()
            raise DeviceError(f"CUDA IPC mapping failed: {next(e for e in errs if e is not None)}")

    def close(self):
        for ptr, o in self.opened:
            _lib.check(_lib.lib().bw_ipc_close_handle(ptr, o))
        self.opened = []


class NarrowWire:
    """Reusable state of the narrow-wire exchange on one rank: the packed
    shard, the overflow flag and the IPC map of every rank's packed shard."""

    def __init__(self, local: torch.Tensor, group, dist):
        self.packed = torch.empty(local.numel() * WIRE_BYTES, dtype=torch.int8, device=local.device)
        self.flag = torch.zeros(1, dtype=torch.int32, device=local.device)
        self.peers = _PeerMap(self.packed, group, dist)

    def close(self):
        self.peers.close()


def narrow_step(local: torch.Tensor, nw: NarrowWire, group, dist, p: int, device_barrier=None, mark=None) -> bool:
    """The narrow-wire transform of this rank's shard (every rank calls it).
    Returns False, with the shard untouched, when some input is too large for
    the wire (the caller then runs the int64 path).  mark(i), if given, is
    called at the phase boundaries (0: start, 1: packed and agreed, 2:
    exchanged, 3: transformed) -- the benchmark records CUDA events there."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mark = mark or (lambda i: None)
    mark(0)
    nw.flag.zero_()
    _pack(local, nw.packed, nw.flag, p)
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(nw.flag, op=dist.ReduceOp.MAX, group=group)  # also barrier (i): every pack is done
        bad = int(nw.flag.item())
    else:
        f = nw.flag.cpu()
        dist.all_reduce(f, op=dist.ReduceOp.MAX, group=group)
        bad = int(f.item())
    if bad:
        return False
    mark(1)
    m = local.numel() // world
    _xshard_narrow(nw.peers.ptrs, p, rank * m, m, local.device)
    if device_barrier is not None:
        device_barrier()
    else:
        torch.cuda.current_stream(local.device).synchronize()
        dist.barrier(group)  # (ii) every slice exchanged before anyone widens
    mark(2)
    _widen(nw.packed, local)
    mark(3)
    return True


last_exchange = None  # the exchange the last fwht_distributed call actually ran (diagnostics)
last_exchanges: list = []  # the exchange of every signal of the last fwht_distributed_many call


def fwht_distributed(local: torch.Tensor, group=None, mode: str = "fused", backend=None,
                     peer_map: _PeerMap | None = None, narrow_wire: NarrowWire | None = None) -> int:
    """Rank r holds shard r (indices r*2**(n-p) ... of a 2**n signal).
    Transforms the whole signal in place across the group; returns
    n * 2**(n-1).  Must be called by every rank of ``group``.

    mode="fused" (default): local passes over the low bits, then K6' (the
    last local pass and the cross-shard stages in one kernel over peer
    pointers); shards under 2**14 points use mode="peer".  mode="narrow":
    the int8 exchange first, then the local transforms (module docstring);
    falls back to "fused" for inputs above 127 >> log2 P.  mode="peer": full
    local transform, then K6 over peer pointers.  mode="a2a": full local
    transform, then all-to-all + K6 on the received slots + all-to-all."""
    import torch.distributed as dist

    global last_exchange
    last_exchange = None
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    p = log2_shards(world)
    backend = backend or CudaBackend()
    local_len = local.numel()
    n_local = local_len.bit_length() - 1
    n = n_local + p
    if mode == "narrow":
        if p > 0 and local.is_cuda and narrow_ok(local_len, p):
            nw = narrow_wire or NarrowWire(local, group, dist)
            done = narrow_step(local, nw, group, dist, p)
            if narrow_wire is None:  # barrier (ii) passed: no peer touches our packed shard any more
                torch.cuda.current_stream(local.device).synchronize()
                nw.close()
            if done:
                last_exchange = "narrow"
                return n << (n - 1)
        mode = "fused"
    if mode == "fused" and p > 0 and n_local >= 14:
        if not local.is_cuda:
            raise BadArguments("mode='fused' needs CUDA shards")
        widths, r = fused_plan(n_local, p)
        _local_partial(local, n_local, widths)
        pm = peer_map or _PeerMap(local, group, dist)
        backend.sync(local)
        dist.barrier(group)  # (i) every shard's local passes are done
        _fused_pass(pm.ptrs, p, n_local, r, rank, local.device)
        backend.sync(local)
        dist.barrier(group)  # (ii) every fused pass is done
        if peer_map is None:
            pm.close()
        last_exchange = "fused"
        return n << (n - 1)
    if mode == "fused":
        mode = "peer"
    backend.local_fwht(local)  # parallel.py phase 0
    if p == 0:
        return n << max(n - 1, 0)
    if mode == "peer":
        if not local.is_cuda:
            raise BadArguments("mode='peer' needs CUDA shards")
        pm = peer_map or _PeerMap(local, group, dist)
        backend.sync(local)
        dist.barrier(group)  # (i) every shard's local passes are done
        b, c = slice_of(rank, world, local_len)
        ptrs = (ctypes.c_void_p * world)(*pm.ptrs)
        with torch.cuda.device(local.device):
            _lib.check(_lib.lib().bw_xshard_i64(ptrs, p, b, c, _stream_handle(local)))
        backend.sync(local)
        dist.barrier(group)  # (ii) every exchange is done before anyone reads
        if peer_map is None:
            pm.close()
        last_exchange = "peer"
        return n << (n - 1)
    if mode == "a2a":
        if local_len % world:
            raise BadArguments("local length must be divisible by the world size")
        m = local_len // world
        recv = torch.empty_like(local)
        dist.all_to_all_single(recv, local, group=group)  # slot r = shard r's slice `rank`
        backend.xshard_slots(recv.view(world, m), p)
        dist.all_to_all_single(local, recv, group=group)
        last_exchange = "a2a"
        return n << (n - 1)
    raise BadArguments(f"unknown mode {mode!r}")


def fwht_distributed_extract_ge(local: torch.Tensor, tau: int, group=None, mode: str = "fused",
                                cap: int = 1 << 16, peer_map: _PeerMap | None = None):
    """fwht_distributed, then every coefficient of the WHOLE 2**n signal with
    |W| >= tau (noisy.py:185-222), as (index, value) CUDA tensors sorted by
    index, on every rank (configs 3/5 over P GPUs).  Must be called by every
    rank of ``group``.

    mode="fused": the threshold test runs on the fused cross-shard pass's
    final values (kernel K6' with the extraction epilogue): each rank's tiles
    span every shard, so its hits carry global indices and are unordered.
    Other modes: the exchange, then the ordered extraction of this rank's own
    shard (indices offset by the shard base).  Either way the ranks' lists
    are gathered (all_gather_object: a few thousand pairs at most) and
    merged by index."""
    import torch.distributed as dist

    global last_exchange
    if tau < 0:
        raise BadArguments(f"tau must be >= 0, got {tau}")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    p = log2_shards(world)
    if not (local.is_cuda and local.dtype == torch.int64 and local.is_contiguous()):
        raise BadArguments("fwht_distributed_extract needs a contiguous CUDA int64 shard")
    n_local = local.numel().bit_length() - 1
    idx = torch.empty(cap, dtype=torch.int64, device=local.device)
    val = torch.empty(cap, dtype=torch.int64, device=local.device)
    if mode == "fused" and p > 0 and n_local >= 14:
        widths, r = fused_plan(n_local, p)
        _local_partial(local, n_local, widths)
        pm = peer_map or _PeerMap(local, group, dist)
        torch.cuda.current_stream(local.device).synchronize()
        dist.barrier(group)  # (i) every shard's local passes are done
        count = torch.zeros(1, dtype=torch.int64, device=local.device)
        _fused_pass_extract(pm.ptrs, p, n_local, r, rank, local.device, int(tau), idx, val, count)
        torch.cuda.current_stream(local.device).synchronize()
        dist.barrier(group)  # (ii) every fused pass is done
        if peer_map is None:
            pm.close()
        k = int(count.item())
        last_exchange = "fused"
    else:
        from .extract import extract_ge

        fwht_distributed(local, group=group, mode=mode, peer_map=peer_map)
        i2, v2 = extract_ge(local, int(tau), base=rank << n_local, cap=cap)
        k = int(i2.numel())
        idx[:k] = i2
        val[:k] = v2
    if k > cap:
        raise BadArguments(f"{k} hits on rank {rank} exceed the capacity {cap}")
    mine = list(zip(idx[:k].tolist(), val[:k].tolist()))
    every = [None] * world
    dist.all_gather_object(every, mine, group=group)
    hits = sorted(h for part in every for h in part)
    out_i = torch.tensor([h[0] for h in hits], dtype=torch.int64, device=local.device)
    out_v = torch.tensor([h[1] for h in hits], dtype=torch.int64, device=local.device)
    return out_i, out_v


def fwht_distributed_extract_gt(local: torch.Tensor, tau: int, group=None, mode: str = "fused", **kw):
    """Config semantics (BASELINE configs 3/5): |W| > tau, sorted by index."""
    return fwht_distributed_extract_ge(local, int(tau) + 1, group=group, mode=mode, **kw)


def fwht_distributed_many(hosts: list, group=None, mode: str = "fused", work=None, peer_maps=None,
                          narrow_wires=None) -> int:
    """fwht_distributed on a sequence of host shards (this rank's pinned
    torch CPU tensors, one per signal; every rank calls it with the same
    count): each is copied in, transformed across the group and copied back
    in place.  The signals alternate between two device buffers, so one
    signal's host->device copy overlaps the previous signal's device->host
    copy (PCIe full duplex), as bw_fwht_host_batch_i64 does on one GPU.
    work / peer_maps / narrow_wires: optional reusable per-buffer state (two
    of each).  Returns n * 2**(n-1) per signal."""
    import torch.distributed as dist

    global last_exchanges
    last_exchanges = []
    if not hosts:
        return 0
    m = hosts[0].numel()
    dev = torch.device("cuda", torch.cuda.current_device())
    work = work or [torch.empty(m, dtype=torch.int64, device=dev) for _ in range(2)]
    own_maps = peer_maps is None and mode in ("fused", "peer")
    if own_maps:
        peer_maps = [_PeerMap(w, group, dist) for w in work]
    peer_maps = peer_maps or [None, None]
    narrow_wires = narrow_wires or [None, None]
    cur = torch.cuda.current_stream(dev)
    up, down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    loaded = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    freed = [torch.cuda.Event() for _ in range(2)]
    up.wait_stream(cur)
    bf = 0
    for i, h in enumerate(hosts):
        b = i & 1
        with torch.cuda.stream(up):
            if i >= 2:
                up.wait_event(freed[b])  # signal i-2's copy-out left this buffer
            if i > 0 and h.data_ptr() == hosts[i - 1].data_ptr():
                up.wait_event(freed[b ^ 1])  # the same host shard twice in a row: in order
            work[b].copy_(h, non_blocking=True)
            loaded[b].record(up)
        cur.wait_event(loaded[b])
        bf = fwht_distributed(work[b], group=group, mode=mode, peer_map=peer_maps[b],
                              narrow_wire=narrow_wires[b])
        last_exchanges.append(last_exchange)
        done[b].record(cur)
        with torch.cuda.stream(down):
            down.wait_event(done[b])
            h.copy_(work[b], non_blocking=True)
            freed[b].record(down)
    cur.wait_stream(down)
    cur.synchronize()
    if own_maps:
        dist.barrier(group)  # every rank's exchanges are done before the mappings close
        for pm in peer_maps:
            pm.close()
    return bf
