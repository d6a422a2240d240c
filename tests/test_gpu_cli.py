"""Experiment driver on the GPU against the reference's own driver: the
configs in tests/golden/cli_runs.json were run through pintlab.cli
(tests/golden/gen_golden_cli.py); the same configs through
paper_2110_10762_b200.cli must give the same rows (iterations, events, stop
reasons, model costs, fitted overhead) and errors / contraction factors
within the stated tolerances."""
import csv
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

with open(os.path.join(GOLDEN, "cli_runs.json"), encoding="utf-8") as _fh:
    RUNS = json.load(_fh)


def _rows(out):
    with open(os.path.join(out, "summary.csv"), newline="", encoding="utf-8") as fh:
        return list(csv.DictReader(fh))


@pytest.mark.parametrize("name", sorted(RUNS))
def test_cli_matches_reference_driver(gpu, tmp_path, name):
    from paper_2110_10762_b200.cli import SUMMARY_COLUMNS, main
    ref = RUNS[name]
    cfg_path = tmp_path / "c.json"
    cfg_path.write_text(json.dumps(ref["config"]), encoding="utf-8")
    out = tmp_path / "out"
    rc = main(["run", "--config", str(cfg_path), "--out", str(out), "--traces"])
    assert rc == ref["exit_code"]
    rows = _rows(out)
    assert list(rows[0].keys()) == SUMMARY_COLUMNS
    assert len(rows) == len(ref["rows"])
    for got, want in zip(rows, ref["rows"]):
        for col in ("label", "p", "mode", "policy", "seed", "delay_bound", "iterations", "events", "stop_reason",
                    "model_cost"):
            assert got[col] == want[col], (col, got, want)
        if want["fitted_overhead"]:
            assert float(got["fitted_overhead"]) == pytest.approx(float(want["fitted_overhead"]), rel=1e-12)
        else:
            assert got["fitted_overhead"] == ""
        # both drivers' errors are against their own sequential fine solve
        assert abs(float(got["error_vs_oracle"]) - float(want["error_vs_oracle"])) < 1e-9
        for col in ("sync_factor", "async_factor"):
            assert float(got[col]) == pytest.approx(float(want[col]), rel=1e-7, abs=1e-12)
        for col in ("sync_margin", "async_margin"):
            assert float(got[col]) == pytest.approx(float(want[col]), abs=1e-7)
    report = json.loads((out / "report.json").read_text(encoding="utf-8"))
    sync = [r for r in report["runs"] if r["mode"] == "sync"][0]
    np.testing.assert_allclose(sync["deltas"], ref["sync_deltas"], rtol=1e-6, atol=1e-13)
    assert report["sequential_cost"] == ref["sequential_cost"]
    assert (out / "traces").is_dir()


def test_cli_device_runs_and_table(gpu, tmp_path):
    from paper_2110_10762_b200.cli import TABLE_COLUMNS, main
    cfg = {"label": "c1", "p": 16, "epsilon": 1e-10,
           "problem": {"name": "heat1d", "n_interior": 1024, "boundary_left": 0.0, "boundary_right": 0.0,
                       "t_final": 1.0, "sine_modes": 8, "seed": 0},
           "fine": {"rule": "backward-euler", "steps": 100}, "coarse": {"rule": "backward-euler", "steps": 1},
           "device_runs": [{"seed": 1}, {"seed": 2, "domains": 4, "delay_frac": 0.1}],
           "measure_costs": True}
    cfg_path = tmp_path / "c.json"
    cfg_path.write_text(json.dumps(cfg), encoding="utf-8")
    out = tmp_path / "out"
    assert main(["run", "--config", str(cfg_path), "--out", str(out)]) == 0
    rows = _rows(out)
    assert [r["mode"] for r in rows] == ["sequential", "sync", "async-device", "async-device"]
    assert rows[1]["iterations"] == "14" and rows[1]["stop_reason"] == "threshold"  # reference C1 k (golden c1_sync)
    for r in rows[2:]:
        assert r["stop_reason"] == "converged" and float(r["error_vs_oracle"]) < 1e-8
        assert int(r["iterations"]) >= 14
    report = json.loads((out / "report.json").read_text(encoding="utf-8"))
    assert report["costs"]["unit"] == "seconds" and report["costs"]["fine_cost"] > 0
    assert all(r["audit"]["ok"] for r in report["runs"] if r["mode"] == "async-device")
    assert main(["table", "--in", str(out / "summary.csv"), "--out", str(tmp_path / "t.csv")]) == 0
    with open(tmp_path / "t.csv", newline="", encoding="utf-8") as fh:
        t = list(csv.DictReader(fh))
    assert list(t[0].keys()) == TABLE_COLUMNS and t[-1]["schedule"] == "device/s2"


def test_cli_3d_config_with_stream_async_runs(gpu, tmp_path):
    """A 3-D configuration through the driver: explicit fine, direct coarse,
    a device async run on CUDA streams with two slice domains."""
    from paper_2110_10762_b200.cli import main
    cfg = {"label": "c4-small", "p": 6, "epsilon": 1e-5, "dtype": "float32", "analysis": False,
           "problem": {"name": "heat3d", "n": 24, "t_final": 6 * 40 * 0.15 / 25 ** 2, "seed": 0},
           "fine": {"rule": "forward-euler", "steps": 40}, "coarse": {"rule": "backward-euler", "steps": 1},
           "device_runs": [{"seed": 3, "domains": 2}]}
    cfg_path = tmp_path / "c.json"
    cfg_path.write_text(json.dumps(cfg), encoding="utf-8")
    out = tmp_path / "out"
    assert main(["run", "--config", str(cfg_path), "--out", str(out)]) == 0
    rows = _rows(out)
    assert [r["mode"] for r in rows] == ["sequential", "sync", "async-device"]
    assert rows[1]["stop_reason"] in ("threshold", "exact") and float(rows[1]["error_vs_oracle"]) < 1e-4
    assert rows[2]["stop_reason"] == "converged" and float(rows[2]["error_vs_oracle"]) < 1e-4
    assert rows[2]["sync_factor"] == ""  # analysis off


def test_cli_runs_are_byte_deterministic(gpu, tmp_path):
    """Reference criterion 11 (test_acceptance.py:380-416, test_cli.py:125-131):
    reruns of a config without device runs or measured costs write
    byte-identical report.json and summary.csv (and traces)."""
    from paper_2110_10762_b200.cli import main
    cfg = RUNS["scalar"]["config"]
    cfg_path = tmp_path / "c.json"
    cfg_path.write_text(json.dumps(cfg), encoding="utf-8")
    outs = []
    for tag in ("a", "b"):
        out = tmp_path / tag
        assert main(["run", "--config", str(cfg_path), "--out", str(out), "--traces"]) == RUNS["scalar"]["exit_code"]
        outs.append(out)
    for name in ("report.json", "summary.csv"):
        assert (outs[0] / name).read_bytes() == (outs[1] / name).read_bytes(), name
    ta = sorted(p.name for p in (outs[0] / "traces").iterdir())
    assert ta == sorted(p.name for p in (outs[1] / "traces").iterdir()) and ta
    for name in ta:
        assert (outs[0] / "traces" / name).read_bytes() == (outs[1] / "traces" / name).read_bytes(), name
