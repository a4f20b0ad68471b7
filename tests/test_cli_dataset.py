"""Dataset format + CLI on the GPU engine (cli.py:144-291, dataset.py:1-88).

CPU: format compatibility with a payload + sidecar written by the reference
itself (tests/golden/ref_dataset_n8.bin), validation errors and exit codes.
GPU: gen-config -> transform mem / transform ext -> extract, end to end
(the reference's acceptance criterion 11, test_acceptance.py:279-340)."""

import json
import os
import shutil

import numpy as np
import pytest

from paper_1607_01039_b200 import cli, dataset
from oracle import oracle_np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def copy_ref_dataset(tmp_path):
    dst = str(tmp_path / "ref.bin")
    shutil.copy(os.path.join(GOLDEN, "ref_dataset_n8.bin"), dst)
    shutil.copy(os.path.join(GOLDEN, "ref_dataset_n8.bin.meta.json"), dst + ".meta.json")
    return dst


def test_reads_reference_dataset(tmp_path):
    path = copy_ref_dataset(tmp_path)
    arr, kind, domain = dataset.read_signal(path)
    assert (kind, domain) == ("int64", "time")
    assert np.array_equal(arr, oracle_np.gen(2, 8, [1000], 0, 1 << 8))


def test_writes_reference_format(tmp_path):
    x = oracle_np.gen(2, 8, [1000], 0, 1 << 8)
    path = str(tmp_path / "ours.bin")
    dataset.write_signal(path, x)
    with open(path, "rb") as a, open(os.path.join(GOLDEN, "ref_dataset_n8.bin"), "rb") as b:
        assert a.read() == b.read()
    with open(path + ".meta.json") as a, open(os.path.join(GOLDEN, "ref_dataset_n8.bin.meta.json")) as b:
        assert json.load(a) == json.load(b)


def test_validation_errors(tmp_path):
    path = copy_ref_dataset(tmp_path)
    with pytest.raises(dataset.PathExists):
        dataset.write_signal(path, np.zeros(4, dtype=np.int64))
    with open(path, "ab") as f:
        f.write(b"\0" * 8)
    with pytest.raises(dataset.SizeMismatch):
        dataset.read_meta(path)
    with pytest.raises(dataset.BadMetadata):
        dataset.read_meta(str(tmp_path / "missing.bin"))
    bad = str(tmp_path / "bad.bin")
    np.zeros(4, dtype="<i8").tofile(bad)
    with open(bad + ".meta.json", "w") as f:
        json.dump({"format_version": 1, "log2_dim": 2, "element_kind": "int32", "domain": "time"}, f)
    with pytest.raises(dataset.BadMetadata):
        dataset.read_meta(bad)


def test_cli_exit_codes(tmp_path, capsys):
    assert cli.run([]) == 1
    assert cli.run(["transform"]) == 1
    assert cli.run(["extract", "--in", "x"]) == 1  # missing --threshold
    assert cli.run(["transform", "mem", "--in", str(tmp_path / "missing.bin")]) == 3  # BadMetadata
    path = copy_ref_dataset(tmp_path)
    dataset.set_domain(path, "walsh")
    assert cli.run(["transform", "mem", "--in", path]) == 3  # already Walsh (BadArguments)


@pytest.mark.gpu
def test_cli_end_to_end(tmp_path, coracle, capsys):
    n = 18
    src = str(tmp_path / "sig.bin")
    assert cli.run(["--quiet", "gen-config", "--config", "3", "--n", str(n), "--out", src]) == 0
    x, _, _ = dataset.read_signal(src)
    ref = x.copy()
    coracle.oracle_fwht_i64(ref.ctypes.data, n)
    ext = str(tmp_path / "ext.bin")
    shutil.copy(src, ext)
    shutil.copy(src + ".meta.json", ext + ".meta.json")
    assert cli.run(["--quiet", "transform", "mem", "--in", src]) == 0
    assert cli.run(["--quiet", "transform", "ext", "--in", ext, "--mem-log2", "15"]) == 0
    for p in (src, ext):
        y, kind, domain = dataset.read_signal(p)
        assert domain == "walsh" and np.array_equal(y, ref)
    capsys.readouterr()
    from paper_1607_01039_b200 import signals

    tau = (1 << 26) >> (30 - n)
    assert cli.run(["--json", "extract", "--in", src, "--threshold", str(tau + 1), "--block-log2", "15"]) == 0
    doc = json.loads(capsys.readouterr().out)
    want = oracle_np.extract_above(ref, tau + 1)
    assert doc["count"] == len(want)
    assert [(c["index"], c["coefficient"]) for c in doc["coefficients"]] == want
    assert [c["index"] for c in doc["coefficients"]] == signals.config(3, n).masks
    assert cli.run(["extract", "--in", src, "--threshold", "1000"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "index,coefficient"
    assert [tuple(map(int, ln.split(","))) for ln in lines[1:]] == oracle_np.extract_above(ref, 1000)


def test_cli_drop_in_options_and_errors(tmp_path, capsys):
    """Options of the reference CLI (cli.py:41-84, 144-257, 477-518) that
    fail before any device work."""
    path = copy_ref_dataset(tmp_path)
    assert cli.run(["transform", "ext", "--in", path, "-b", "20", "--resume"]) == 3
    assert cli.run(["transform", "ext", "--in", path, "-b", "20", "--io-block-bytes", "12"]) == 3
    assert cli.run(["transform", "ext", "--in", path, "-b", "20", "--mode", "sideways"]) == 1
    assert cli.run(["oracle", "--in", path]) == 1  # needs --out and/or --expect
    assert cli.run(["transform", "mem", "--in", path, "--threads", "3"]) == 3  # InvalidWorkerCount
    bare = str(tmp_path / "bare.bin")
    np.arange(16, dtype="<i8").tofile(bare)
    assert cli.run(["transform", "mem", "--in", bare]) == 3  # no sidecar, no --force
    assert dataset.adopt(bare, "int64", "time") == 4
    with pytest.raises(dataset.PathExists):
        dataset.adopt(bare, "int64", "time")
    odd = str(tmp_path / "odd.bin")
    np.arange(3, dtype="<i8").tofile(odd)
    with pytest.raises(dataset.SizeMismatch):
        dataset.adopt(odd, "int64", "time")


def test_map_file_format(tmp_path, golden_npz):
    """subspace.py:288-310: d_out lines of d_in '0'/'1' chars, bit 0 first."""
    from paper_1607_01039_b200 import subspace

    z = golden_npz("fold_16_8.npz")
    path = str(tmp_path / "m.txt")
    subspace.save_map(z["rows"], path)
    lines = open(path).read().splitlines()
    assert len(lines) == 8 and all(len(ln) == 16 for ln in lines)
    assert lines[0] == "".join(str(int(v)) for v in z["rows"][0])
    assert np.array_equal(subspace.load_map(path), z["rows"])
    with open(path, "a") as f:
        f.write("0120\n")
    with pytest.raises(dataset.BadMetadata):
        subspace.load_map(path)


@pytest.mark.gpu
def test_cli_oracle_fold_threads_and_float_extract(tmp_path, coracle, golden_npz, capsys):
    # transform mem --threads 4: the run_parallel schedule on the GPU
    n = 16
    x = oracle_np.gen(2, 41, [1 << 20], 0, 1 << n)
    src = str(tmp_path / "t.bin")
    dataset.write_signal(src, x)
    assert cli.run(["--quiet", "transform", "mem", "--in", src, "--threads", "4"]) == 0
    ref = x.copy()
    coracle.oracle_fwht_i64(ref.ctypes.data, n)
    y, _, domain = dataset.read_signal(src)
    assert domain == "walsh" and np.array_equal(y, ref)
    # oracle --out / --expect
    small = str(tmp_path / "s.bin")
    xs = oracle_np.gen(2, 42, [1 << 10], 0, 1 << 10)
    dataset.write_signal(small, xs)
    out = str(tmp_path / "s_w.bin")
    assert cli.run(["--quiet", "oracle", "--in", small, "--out", out]) == 0
    refs = xs.copy()
    coracle.oracle_fwht_i64(refs.ctypes.data, 10)
    assert np.array_equal(dataset.read_signal(out)[0], refs)
    capsys.readouterr()
    assert cli.run(["oracle", "--in", small, "--expect", out]) == 0
    assert capsys.readouterr().out.strip() == "match"
    wrong = str(tmp_path / "wrong.bin")
    refs[3] += 1
    dataset.write_signal(wrong, refs, domain="walsh")
    assert cli.run(["oracle", "--in", small, "--expect", wrong]) == 3
    # fold --gen-dout: the map and the folded signal equal the reference's (golden)
    z = golden_npz("fold_16_8.npz")
    fsrc = str(tmp_path / "f.bin")
    dataset.write_signal(fsrc, oracle_np.gen(1, 77, [], 0, 1 << 16))
    m = str(tmp_path / "m.txt")
    fout = str(tmp_path / "folded.bin")
    assert cli.run(["--quiet", "fold", "--in", fsrc, "--matrix", m, "--out", fout, "--gen-dout", "8",
                    "--seed", "7"]) == 0
    from paper_1607_01039_b200 import subspace

    assert np.array_equal(subspace.load_map(m), z["rows"])
    assert np.array_equal(dataset.read_signal(fout)[0], z["folded"])
    assert cli.run(["fold", "--in", fsrc, "--matrix", m, "--out", str(tmp_path / "f2.bin"), "--gen-dout", "8"]) == 3
    # extract on a float64 Walsh-domain dataset (noisy.py:217-222 float values)
    rng = np.random.default_rng(5)
    w = rng.normal(scale=100.0, size=1 << 12)
    wpath = str(tmp_path / "w.bin")
    dataset.write_signal(wpath, w, domain="walsh")
    capsys.readouterr()
    assert cli.run(["--json", "extract", "--in", wpath, "--threshold", "180.5"]) == 0
    doc = json.loads(capsys.readouterr().out)
    assert [(c["index"], c["coefficient"]) for c in doc["coefficients"]] == oracle_np.extract_above(w, 180.5)


def test_cli_ext_refuses_interrupted_reference_run(tmp_path, capsys):
    """A sidecar carrying the reference executor's pass-progress marker
    (an interrupted `transform ext`, external.py:155-178) is refused with the
    reference's messages, before any device work; the payload is untouched."""
    path = copy_ref_dataset(tmp_path)
    before = open(path, "rb").read()
    meta = dataset.read_meta(path)
    marker = {"mode": "blocked", "mem_log2": 6, "io_block_elems": 8, "passes_done": 1, "total_passes": 3,
              "writing": False}
    for writing, resume, needle in ((False, False, "has an interrupted transform (1/3 passes done)"),
                                    (True, False, "has an interrupted transform (1/3 passes done)"),
                                    (True, True, "was interrupted after its writes began"),
                                    (False, True, "cannot resume")):
        meta["pass_progress"] = dict(marker, writing=writing)
        with open(path + ".meta.json", "w") as f:
            json.dump(meta, f)
        capsys.readouterr()
        argv = ["transform", "ext", "--in", path, "-b", "6"] + (["--resume"] if resume else [])
        assert cli.run(argv) == 3
        assert needle in capsys.readouterr().err
        assert open(path, "rb").read() == before
        assert dataset.read_meta(path)["domain"] == "time"
