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

Three drivers share that kernel:
  * ``fwht_shards``      -- one process, shards on one or several devices
                            (single-GPU P-shard emulation, or P2P over NVLink).
  * ``fwht_distributed`` -- one process per GPU (torch.distributed):
      mode="peer": CUDA IPC peer pointers, the K6 kernel reads and writes the
                   peers' HBM directly over NVLink (fused compute+exchange);
      mode="a2a":  all-to-all transpose + local K6 on the receive slots +
                   all-to-all back (NCCL on GPUs; gloo on CPU for tests).
"""

from __future__ import annotations

import ctypes
import json

import torch

from . import _lib
from .core import _is_power_of_two, _stream_handle, fwht_array
from .errors import BadArguments, InvalidWorkerCount


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


def fwht_shards(shards: list[torch.Tensor]) -> int:
    """Transform the 2**n signal whose P = len(shards) contiguous shards are
    given (shard r = indices r*2**(n-p) ...), in place.  Shards may live on
    one device (emulation of P GPUs) or on P devices (P2P over NVLink).
    Returns n * 2**(n-1)."""
    p = log2_shards(len(shards))
    local = shards[0].numel()
    for s in shards:
        if s.numel() != local or s.dtype != torch.int64 or not s.is_cuda or not s.is_contiguous():
            raise BadArguments("shards must be equal-length contiguous CUDA int64 tensors")
    n_local = local.bit_length() - 1
    for s in shards:  # parallel.py phase 0: independent local transforms
        with torch.cuda.device(s.device):
            fwht_array(s)
    if p == 0:
        return (n_local) << max(n_local - 1, 0)
    devices = sorted({s.device.index for s in shards})
    if len(devices) > 1:
        for d in devices:  # barrier (i): every local transform done
            torch.cuda.synchronize(d)
        for d in devices:
            with torch.cuda.device(d):
                for q in devices:
                    _lib.check(_lib.lib().bw_enable_peer_access(q))
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
        torch.cuda.synchronize(t.device)


class _PeerMap:
    """CUDA IPC mapping of every rank's shard into this process."""

    def __init__(self, local: torch.Tensor, group, dist):
        L = _lib.lib()
        handle = (ctypes.c_char * 64)()
        off = ctypes.c_uint64(0)
        _lib.check(L.bw_ipc_get_handle(local.data_ptr(), handle, ctypes.byref(off)))
        mine = (bytes(handle), int(off.value))
        world = dist.get_world_size(group)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        self.rank = dist.get_rank(group)
        self.ptrs, self.opened = [], []
        for r, (h, o) in enumerate(allh):
            if r == self.rank:
                self.ptrs.append(local.data_ptr())
                continue
            ptr = ctypes.c_void_p(0)
            _lib.check(L.bw_ipc_open_handle(h, o, ctypes.byref(ptr)))
            self.ptrs.append(ptr.value)
            self.opened.append((ptr.value, o))

    def close(self):
        for ptr, o in self.opened:
            _lib.check(_lib.lib().bw_ipc_close_handle(ptr, o))
        self.opened = []


def fwht_distributed(local: torch.Tensor, group=None, mode: str = "peer", backend=None,
                     peer_map: _PeerMap | None = None) -> int:
    """Rank r holds shard r (indices r*2**(n-p) ... of a 2**n signal).
    Transforms the whole signal in place across the group; returns
    n * 2**(n-1).  Must be called by every rank of ``group``."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    p = log2_shards(world)
    backend = backend or CudaBackend()
    local_len = local.numel()
    n_local = local_len.bit_length() - 1
    backend.local_fwht(local)  # parallel.py phase 0
    n = n_local + p
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
        return n << (n - 1)
    if mode == "a2a":
        if local_len % world:
            raise BadArguments("local length must be divisible by the world size")
        m = local_len // world
        recv = torch.empty_like(local)
        dist.all_to_all_single(recv, local, group=group)  # slot r = shard r's slice `rank`
        backend.xshard_slots(recv.view(world, m), p)
        dist.all_to_all_single(local, recv, group=group)
        return n << (n - 1)
    raise BadArguments(f"unknown mode {mode!r}")
