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
