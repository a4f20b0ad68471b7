"""bench.py contract: one JSON line with the driver's keys."""

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port() -> str:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return str(port)


def run_bench(args, env=None, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, env={**os.environ, **(env or {})}, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run_bench(["--impl", "reference", "--steps", "1", "--warmup", "0", "--log2n", "18"])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    shipped = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "bigwht"))
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == ("reference" if shipped else "port")
    assert d["config"]["workload"].startswith("config4")
    if shipped:
        assert "bigwht.parallel.run_parallel" in d["cpu_baseline"]["sample"]


def test_reference_arm_full_size_run():
    """--cpu-full: one run of the reference at the full (here small) size,
    reported beside the extrapolated sample rate."""
    d = run_bench(["--impl", "reference", "--steps", "1", "--warmup", "0", "--log2n", "16", "--cpu-full"])
    full = d["cpu_baseline"]["full_size_measured"]
    assert full["n"] == 16 and full["seconds"] > 0 and full["points_per_s"] > 0


@pytest.mark.gpu
def test_ours_contract_small():
    d = run_bench(["--steps", "3", "--warmup", "3", "--log2n", "24", "--no-cpu"])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "dtype", "config",
                "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["roofline"]["bound"] == "hbm" and d["roofline"]["peak"] > 0
    assert d["gpu_launches"] == 3 * len(d["config"]["passes"])
    assert d["e2e"]["h2d_bytes_per_step"] == 8 << 24
    ep = d["entry_points"]  # fwht_inplace beside fwht_array (core.py:120-125)
    assert ep["max_abs"] == 1 and ep["fwht_inplace_ms"] > 0 and ep["fwht_inplace_known_bound_ms"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("config,n", [(4, 24), (3, 24), (2, 22)])
def test_ours_parity_in_the_bench_line(config, n):
    """The CPU baseline leg runs the reference (baseline/_ref when shipped)
    on a sample; the same run checks it bit-exactly against the GPU, and
    checks the measured step's own full-size output by the fold spot check."""
    d = run_bench(["--config", str(config), "--steps", "3", "--warmup", "3", "--log2n", str(n), "--no-e2e"])
    par = d["parity"]
    assert par["equal"] is True, par
    assert par["sample"]["equal"] and par["sample"]["points"] == 1 << n
    assert par["full_size_spot_check"]["equal"] and par["full_size_spot_check"]["points"] == 1 << 20
    assert d["cpu_baseline"]["value"] > 0


@pytest.mark.gpu
def test_multirank_path_two_processes_one_gpu():
    """The N > 1 bench path (CUDA-IPC peer exchange, max over ranks, rank-0
    JSON) with 2 ranks on one GPU; gloo carries the host-side collectives."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", free_port(), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--log2n", "24", "--dist-backend", "gloo", "--no-cpu"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["log2p"] == 1 and "nvlink" in d and d["value"] > 0


@pytest.mark.gpu
def test_multirank_narrow_wire_two_processes_one_gpu():
    """bench --mode narrow: the int8 cross-first exchange, timed by phase,
    with no fallback on config 4's +-1 signal."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", free_port(), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--log2n", "24", "--dist-backend", "gloo", "--no-cpu",
           "--mode", "narrow"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    assert d["config"]["exchange"] == "narrow" and d["config"]["passes"]["fallbacks_to_int64"] == 0
    assert set(d["passes_ms"]) == {"pack_and_agree", "exchange", "local_transform"}
    assert d["nvlink"]["bytes_each_direction"] == (1 << 23) / 2
    assert "narrow x2" in d["e2e"]["api"] and "fused" not in d["e2e"]["api"], d["e2e"]["api"]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["fused", "narrow"])
def test_multirank_extraction_config3_two_processes_one_gpu(mode):
    """Config 3 on 2 ranks: the extraction fused into the cross-shard pass
    (fused) or run on every rank's shard after the exchange (narrow), inside
    the step; the gathered hits are the planted secret."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", free_port(),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "3", "--steps", "3", "--warmup", "3",
           "--dist-backend", "gloo", "--no-cpu", "--no-e2e", "--mode", mode]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    assert d["extraction"]["recovered_planted"] is True, d["extraction"]
    assert ("cross-shard pass" if mode == "fused" else "after the exchange") in d["extraction"]["rule"]


@pytest.mark.gpu
def test_narrow_intermediates_bench_leg():
    d = run_bench(["--steps", "3", "--warmup", "3", "--log2n", "26", "--no-cpu", "--no-e2e",
                   "--intermediates", "narrow"])
    assert d["config"]["narrow_fallbacks"] == 0 and d["config"]["algorithmic_bytes_per_point"] == [10, 6, 12]
    assert d["roofline"]["kernel"].startswith("narrow pass") and "flag_readback_ms" in d


@pytest.mark.gpu
def test_compact_intermediates_bench_leg():
    """--intermediates compact at a small size: the first pass checked inside
    the step, no fallback on the +-1 config input, 12 / 8 / 12 bytes per point,
    and the in-run parity of the measured step."""
    d = run_bench(["--steps", "3", "--warmup", "3", "--log2n", "24", "--no-e2e", "--intermediates", "compact"])
    assert d["config"]["compact_fallbacks"] == 0 and d["config"]["algorithmic_bytes_per_point"] == [12, 8, 12]
    assert d["roofline"]["kernel"].startswith("compact pass") and "flag_readback_ms" in d
    assert d["gpu_launches"] == 3 * 3
    assert d["parity"]["equal"] is True


@pytest.mark.gpu
def test_default_bench_runs_the_compact_plan_where_the_library_does():
    """n = 30: the library's default (bw_compact_auto) is the compact plan on
    the int32 engine, so the default bench line measures it; config 2's
    wide inputs at the same size run the int64 plan after the restore."""
    d = run_bench(["--steps", "3", "--warmup", "3", "--log2n", "30", "--no-e2e", "--no-cpu"])
    assert d["config"]["compact_fallbacks"] == 0
    assert [q["bytes_per_point"] for q in d["config"]["passes"]] == [12, 8, 12]
    assert all(q["kernel"].startswith("k32_") for q in d["config"]["passes"])
    ep = d["entry_points"]
    assert ep["fwht_array_ran_compact_plan"] is True
    assert ep["fwht_array_ms"] < ep["fwht_array_int64_plan_ms"]
    d = run_bench(["--config", "2", "--steps", "3", "--warmup", "3", "--log2n", "30", "--no-e2e", "--no-cpu",
                   "--no-entry-points"])
    assert d["config"]["compact_fallbacks"] == 6
