"""CLI: verify / simulate / overhead, reference conventions.

Host-only checks run everywhere; the commands that compute are marked gpu.
"""

import csv
import io
import json

import pytest

from paper_2110_03901_b200 import cli
from paper_2110_03901_b200.functional import Method
from paper_2110_03901_b200.lowering import lowered_memory_footprint


def _workload(tmp_path, layers, **extra):
    p = tmp_path / "wl.json"
    p.write_text(json.dumps({"model": "tiny", "layers": layers, **extra}))
    return str(p)


LAYERS = [
    {"name": "a", "n": 2, "c_i": 16, "h_i": 9, "w_i": 7, "c_o": 24, "h_f": 3, "w_f": 3, "stride": 1, "pad": 1},
    {"name": "b", "n": 1, "c_i": 8, "h_i": 12, "w_i": 12, "c_o": 16, "h_f": 5, "w_f": 3, "stride_h": 2,
     "stride_w": 1, "pad_h": 2, "pad_w": 1, "dilation": 2},
]


def _rows(text):
    lines = text.splitlines()
    assert lines[0] == "# sasim-csv v1"
    return list(csv.DictReader(io.StringIO("\n".join(lines[1:]))))


def test_overhead_rows_and_total(tmp_path, capsys):
    path = _workload(tmp_path, LAYERS)
    assert cli.main(["overhead", "--workload", path]) == 0
    rows = _rows(capsys.readouterr().out)
    assert [r["name"] for r in rows] == ["a", "b", "TOTAL"]
    wl = cli.load_workload(path)
    fps = [lowered_memory_footprint(sp, 2) for _, sp in wl["layers"]]
    assert int(rows[0]["lowered_bytes"]) == fps[0]["lowered_bytes"]
    assert int(rows[2]["original_bytes"]) == sum(f["original_bytes"] for f in fps)


def test_workload_schema_and_errors(tmp_path, capsys):
    wl = cli.load_workload(_workload(tmp_path, LAYERS, methods=["cf", "explicit"], seed=7))
    (na, a), (nb, b) = wl["layers"]
    assert (a.stride_h, a.pad_w) == (1, 1)
    assert (b.stride_h, b.stride_w, b.pad_h, b.dilation_w) == (2, 1, 2, 2)
    assert wl["methods"] == [Method.CHANNEL_FIRST_IMPLICIT, Method.EXPLICIT_IM2COL] and wl["seed"] == 7
    bad = [dict(LAYERS[0], stride_h=2)]  # stride and stride_h together
    assert cli.main(["overhead", "--workload", _workload(tmp_path, bad)]) == 2
    assert "error: WorkloadError" in capsys.readouterr().err
    dup = [LAYERS[0], LAYERS[0]]
    assert cli.main(["overhead", "--workload", _workload(tmp_path, dup)]) == 2
    assert "duplicate layer name" in capsys.readouterr().err
    assert cli.main(["overhead", "--workload", str(tmp_path / "missing.json")]) == 2


def test_method_aliases():
    assert Method.parse("channel-first") is Method.CHANNEL_FIRST_IMPLICIT
    assert Method.parse("CL") is Method.CHANNEL_LAST_IMPLICIT
    assert Method.parse("plain_gemm") is Method.PLAIN_GEMM is Method.GEMM
    with pytest.raises(ValueError):
        Method.parse("winograd")


@pytest.mark.gpu
def test_verify_random_cases(capsys):
    """The reference's acceptance criterion c1 (test_acceptance.py:42-57): 200 random specs,
    every method bit-exact against the integer oracle."""
    assert cli.main(["verify", "--count", "200", "--seed", "20240001"]) == 0
    assert capsys.readouterr().out.strip() == "200/200 match"


@pytest.mark.gpu
def test_simulate_verify_rows(tmp_path, capsys):
    path = _workload(tmp_path, LAYERS, methods=["cf", "cl", "explicit"])
    out = tmp_path / "sim.csv"
    assert cli.main(["simulate", "--workload", path, "--verify", "--out", str(out)]) == 0
    rows = _rows(out.read_text())
    assert len(rows) == 6 and all(r["verified"] == "1" and not r["error"] for r in rows)
    assert all(float(r["tflops"]) > 0 and int(r["dram_read_bytes"]) > 0 for r in rows)
    assert capsys.readouterr().out.strip() == "6/6 match"
