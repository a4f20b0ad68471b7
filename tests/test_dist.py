"""Multi-process sharded transform (parallel.py:87-198 with m = P ranks).

* CPU (gloo, world size 2 and 4): the all-to-all orchestration of
  ``sharded.fwht_distributed(mode="a2a")`` with the CPU oracle plugged in as
  the compute backend (test-only), checked against the oracle's full
  transform.
* GPU (one device, 2 processes, gloo for the host barriers): the CUDA-IPC
  peer path -- each process maps the other's shard and runs kernel K6 on its
  own slice in place.  No kernel waits on another, so two ranks on one GPU
  are safe.
"""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleBackend:
    """Test-only compute backend: the CPU oracle on CPU tensors."""

    def __init__(self):
        from oracle import load_c

        self.lib = load_c()

    def local_fwht(self, t):
        a = t.numpy()
        self.lib.oracle_fwht_i64(a.ctypes.data, int(a.size).bit_length() - 1)

    def xshard_slots(self, slots, p):
        rows = slots.numpy()  # [P, m] view, modified in place
        for b in range(p):  # ascending stage order (parallel.py:103-110)
            step = 1 << b
            for r in range(rows.shape[0]):
                if not (r >> b) & 1:
                    a = rows[r].copy()
                    c = rows[r + step].copy()
                    rows[r] = a + c
                    rows[r + step] = a - c

    def sync(self, t):
        pass


def _a2a_worker(rank, world, port, n, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle_np
    from paper_1607_01039_b200 import sharded

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    p = world.bit_length() - 1
    nl = n - p
    x = oracle_np.gen(2, 99, [1 << 20], rank << nl, 1 << nl)
    t = torch.from_numpy(x.copy())
    bf = sharded.fwht_distributed(t, mode="a2a", backend=OracleBackend())
    assert bf == n << (n - 1)
    np.save(os.path.join(out_dir, f"shard{rank}.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_a2a_orchestration_gloo(tmp_path, coracle, world):
    from oracle import oracle_np

    n = 12
    mp.spawn(_a2a_worker, args=(world, free_port(), n, str(tmp_path)), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"shard{r}.npy") for r in range(world)])
    ref = oracle_np.gen(2, 99, [1 << 20], 0, 1 << n)
    coracle.oracle_fwht_i64(ref.ctypes.data, n)
    assert np.array_equal(got, ref)


def _peer_worker(rank, world, port, n, out_dir, mode="peer", kind=2):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle_np
    from paper_1607_01039_b200 import sharded

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    p = world.bit_length() - 1
    nl = n - p
    x = oracle_np.gen(kind, 7, [1 << 20] if kind == 2 else [], rank << nl, 1 << nl)
    t = torch.from_numpy(x).cuda()
    bf = sharded.fwht_distributed(t, mode=mode)
    assert bf == n << (n - 1)
    with open(os.path.join(out_dir, f"mode{rank}.txt"), "w") as f:
        f.write(str(sharded.last_exchange))
    np.save(os.path.join(out_dir, f"shard{rank}.npy"), t.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["peer", "fused"])
def test_peer_ipc_two_processes_one_gpu(tmp_path, coracle, mode):
    from oracle import oracle_np

    n, world = 20, 2
    mp.spawn(_peer_worker, args=(world, free_port(), n, str(tmp_path), mode), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"shard{r}.npy") for r in range(world)])
    ref = oracle_np.gen(2, 7, [1 << 20], 0, 1 << n)
    coracle.oracle_fwht_i64(ref.ctypes.data, n)
    assert np.array_equal(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,expect", [(1, "narrow"), (2, "fused")])
def test_narrow_wire_two_processes_one_gpu(tmp_path, coracle, kind, expect):
    """mode="narrow" over CUDA IPC: a +-1 signal takes the int8 exchange;
    a wide one (|x| up to 2^20) is flagged by the pack kernel and falls back
    to the fused int64 path.  Both equal the oracle."""
    from oracle import oracle_np

    n, world = 20, 2
    mp.spawn(_peer_worker, args=(world, free_port(), n, str(tmp_path), "narrow", kind), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"shard{r}.npy") for r in range(world)])
    ref = oracle_np.gen(kind, 7, [1 << 20] if kind == 2 else [], 0, 1 << n)
    coracle.oracle_fwht_i64(ref.ctypes.data, n)
    assert np.array_equal(got, ref)
    assert [open(tmp_path / f"mode{r}.txt").read() for r in range(world)] == [expect] * world


def _many_worker(rank, world, port, n, out_dir, mode):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle_np
    from paper_1607_01039_b200 import sharded

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    p = world.bit_length() - 1
    nl = n - p
    hosts = [torch.from_numpy(oracle_np.gen(1 + s % 2, 11 + s, [1 << 20] if s % 2 else [], rank << nl, 1 << nl))
             .pin_memory() for s in range(3)]
    order = [hosts[0], hosts[1], hosts[2], hosts[2]]  # the last shard twice in a row: in order
    bf = sharded.fwht_distributed_many(order, mode=mode)
    assert bf == n << (n - 1)
    for s, h in enumerate(hosts):
        np.save(os.path.join(out_dir, f"sig{s}_shard{rank}.npy"), h.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["fused", "narrow", "peer"])
def test_distributed_many_two_processes_one_gpu(tmp_path, coracle, mode):
    """fwht_distributed_many: consecutive host shards through two device
    buffers per rank (H2D of one overlapping D2H of the previous), every
    exchange mode, a shard listed twice in a row (H H x = 2^n x)."""
    from oracle import oracle_np

    n, world = 20, 2
    mp.spawn(_many_worker, args=(world, free_port(), n, str(tmp_path), mode), nprocs=world, join=True)
    for s in range(3):
        got = np.concatenate([np.load(tmp_path / f"sig{s}_shard{r}.npy") for r in range(world)])
        x = oracle_np.gen(1 + s % 2, 11 + s, [1 << 20] if s % 2 else [], 0, 1 << n)
        if s == 2:
            ref = x << n
        else:
            ref = x.copy()
            coracle.oracle_fwht_i64(ref.ctypes.data, n)
        assert np.array_equal(got, ref), s


# ---------------------------------------------- world 4 / 8 on one GPU ---
#
# The N > 1 path at the world sizes of an 8 x B200 box, with every rank on
# the one GPU this build has (gloo for the host barriers, CUDA IPC for the
# peer pointers).  No kernel waits on another kernel (the barriers are host
# side), so co-resident ranks are safe.  Configs 4 (n = 24, +-1) and 5
# (n = 26, 8 planted masks, threshold scaled to 2^29 >> (34 - n)), each
# exchange mode, with the distributed extraction for config 5.

def _cfg_worker(rank, world, port, cfg, n, out_dir, mode):
    import sys

    sys.path.insert(0, ROOT)
    from paper_1607_01039_b200 import sharded, signals

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    p = world.bit_length() - 1
    nl = n - p
    spec = signals.config(cfg, n)
    t = torch.empty(1 << nl, dtype=torch.int64, device="cuda")
    signals.generate(spec, t, base=rank << nl)
    if spec.threshold is not None:
        tau = spec.threshold >> (34 - n)
        i, v = sharded.fwht_distributed_extract_gt(t, tau, mode=mode)
        np.save(os.path.join(out_dir, f"hits{rank}.npy"), np.stack([i.cpu().numpy(), v.cpu().numpy()]))
    else:
        assert sharded.fwht_distributed(t, mode=mode) == n << (n - 1)
    with open(os.path.join(out_dir, f"mode{rank}.txt"), "w") as f:
        f.write(str(sharded.last_exchange))
    np.save(os.path.join(out_dir, f"shard{rank}.npy"), t.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [4, 8])
@pytest.mark.parametrize("cfg,n", [(4, 24), (5, 26)])
@pytest.mark.parametrize("mode", ["fused", "peer", "narrow"])
def test_world_4_8_one_gpu_configs(tmp_path, coracle, world, cfg, n, mode):
    from oracle import oracle_np
    from paper_1607_01039_b200 import signals

    mp.spawn(_cfg_worker, args=(world, free_port(), cfg, n, str(tmp_path), mode), nprocs=world, join=True)
    spec = signals.config(cfg, n)
    ref = oracle_np.gen(spec.kind, spec.seed, list(spec.params), 0, 1 << n)
    coracle.oracle_fwht_i64(ref.ctypes.data, n)
    got = np.concatenate([np.load(tmp_path / f"shard{r}.npy") for r in range(world)])
    assert np.array_equal(got, ref)
    ran = {open(tmp_path / f"mode{r}.txt").read() for r in range(world)}
    assert ran == {mode}, ran  # +-1 and 8-mask inputs both fit the int8 wire at P <= 8
    if spec.threshold is not None:
        tau = spec.threshold >> (34 - n)
        want = oracle_np.extract_gt_by_index(ref, tau)
        for r in range(world):  # every rank holds the whole merged list
            h = np.load(tmp_path / f"hits{r}.npy")
            assert [tuple(map(int, c)) for c in h.T] == [tuple(map(int, w)) for w in zip(*want)]
        assert sorted(int(i) for i in np.load(tmp_path / "hits0.npy")[0]) == sorted(spec.masks)


# ------------------------------------------------ NCCL on the GPU box ---

def _nccl_worker(rank, world, port, out_dir):
    import ctypes as C
    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle_np
    from paper_1607_01039_b200 import _lib, sharded

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    # every NCCL call the bench's N > 1 path makes, in a world-size-1 group
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    ones = torch.ones(1, device="cuda")
    dist.all_reduce(ones)  # the device-side barrier of the timed loop
    torch.cuda.synchronize()
    assert ones.item() == world
    every = [None] * world
    dist.all_gather_object(every, [(rank, 1)])  # the hit gather of configs 3/5
    assert every == [[(0, 1)]]
    t = torch.tensor([1.5], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # the max-over-ranks timing
    results = {}
    for p in (1, 2, 3):  # the a2a exchange: all_to_all_single, K6 on the [P, m] receive rows, back
        P, m = 1 << p, 1 << 12
        x = torch.from_numpy(oracle_np.gen(2, 40 + p, [1 << 20], 0, P * m)).cuda()
        recv = torch.empty_like(x)
        dist.all_to_all_single(recv, x)
        _lib.check(_lib.lib().bw_xshard_strided_i64(recv.data_ptr(), m, p, 0, m,
                                                    torch.cuda.current_stream().cuda_stream))
        dist.all_to_all_single(x, recv)
        rows = oracle_np.gen(2, 40 + p, [1 << 20], 0, P * m).reshape(P, m)
        for b in range(p):  # P-point WHT across the rows (parallel.py:103-110)
            for r in range(P):
                if not (r >> b) & 1:
                    a, c = rows[r].copy(), rows[r + (1 << b)].copy()
                    rows[r], rows[r + (1 << b)] = a + c, a - c
        results[p] = bool(np.array_equal(x.cpu().numpy().reshape(P, m), rows))
    # the public multi-GPU entry points over an NCCL group (P = 1: local transform only)
    y = torch.from_numpy(oracle_np.gen(2, 5, [1 << 20], 0, 1 << 16)).cuda()
    for mode in ("fused", "peer", "a2a", "narrow"):
        z = y.clone()
        sharded.fwht_distributed(z, mode=mode)
        ref = y.cpu().numpy().copy()
        oracle_np.fwht_array(ref)
        results[mode] = bool(np.array_equal(z.cpu().numpy(), ref))
    with open(os.path.join(out_dir, "nccl.txt"), "w") as f:
        f.write(repr(results))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_calls_world_size_one(tmp_path):
    mp.spawn(_nccl_worker, args=(1, free_port(), str(tmp_path)), nprocs=1, join=True)
    res = eval(open(tmp_path / "nccl.txt").read())
    assert res == {1: True, 2: True, 3: True, "fused": True, "peer": True, "a2a": True, "narrow": True}, res
