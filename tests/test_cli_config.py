"""Experiment-driver surface on CPU (reference: pintlab/cli.py and its tests,
test_cli.py:49-200): config validation, exit codes for configuration
errors, config round trip and the condensed table. Runs that touch the GPU
are in test_gpu_cli.py."""
import csv
import json

import pytest

from paper_2110_10762_b200.cli import SUMMARY_COLUMNS, TABLE_COLUMNS, emit_table, load_config, main, parse_config
from paper_2110_10762_b200.errors import ConfigError


def base_config(**overrides):
    cfg = {
        "label": "demo",
        "problem": {"name": "scalar-decay", "rate": 1.0, "t_final": 8.0},
        "p": 8,
        "fine": {"rule": "trapezoidal", "steps": 25},
        "coarse": {"rule": "backward-euler", "steps": 1},
        "epsilon": 1e-5,
        "schedules": [{"seed": 1, "delay_bound": 0, "policy": "round-robin"},
                      {"seed": 2, "delay_bound": 2, "policy": "random-fair"}],
    }
    cfg.update(overrides)
    return cfg


@pytest.mark.parametrize("mutate", [
    lambda c: c.pop("p"),
    lambda c: c.pop("fine"),
    lambda c: c.update(p=0),
    lambda c: c.update(p=True),
    lambda c: c.update(epsilon=-1.0),
    lambda c: c.update(norm="manhattan"),
    lambda c: c.update(mystery=1),
    lambda c: c["problem"].update(name="pendulum"),
    lambda c: c["problem"].update(viscosity=2.0),
    lambda c: c["fine"].update(rule="leapfrog"),
    lambda c: c["fine"].update(steps=0),
    lambda c: c["schedules"].append({"seed": 3, "delay_bound": -1}),
    lambda c: c["schedules"].append({"seed": 3, "delay_bound": 0, "policy": "eager"}),
    lambda c: c.update(costs={"fine_cost": -2.0}),
    lambda c: c.update(k_max=0),
    # B200 extensions
    lambda c: c["fine"].update(dtype="float16"),
    lambda c: c.update(dtype="bf16"),
    lambda c: c["coarse"].update(solver="lu"),
    lambda c: c["fine"].update(tile=4),
    lambda c: c.update(device_runs=[{"domains": 0}]),
    lambda c: c.update(device_runs=[{"domains": 9}]),  # more domains than slices
    lambda c: c.update(device_runs=[{"delay_frac": -0.1}]),
    lambda c: c.update(device_runs=[{"seed": 1, "gpus": 2}]),
    lambda c: c.update(analysis="yes"),
    lambda c: c.update(costs={"fine_cost": True}),
    lambda c: c.update(problem={"name": "heat3d", "n": 8, "viscosity": 1.0}),
])
def test_invalid_configs_rejected(mutate):
    cfg = base_config()
    mutate(cfg)
    with pytest.raises(ConfigError):
        parse_config(cfg)


def test_invalid_config_exits_one(tmp_path, capsys):
    path = tmp_path / "c.json"
    path.write_text(json.dumps(base_config(p=-3)), encoding="utf-8")
    assert main(["run", "--config", str(path), "--out", str(tmp_path / "o")]) == 1
    assert "config error" in capsys.readouterr().err


def test_malformed_and_missing_config_exit_one(tmp_path, capsys):
    bad = tmp_path / "bad.json"
    bad.write_text("{not json", encoding="utf-8")
    assert main(["run", "--config", str(bad), "--out", str(tmp_path / "o")]) == 1
    assert main(["run", "--config", str(tmp_path / "nope.json"), "--out", str(tmp_path / "o")]) == 1


def test_extended_problems_and_round_trip(tmp_path):
    import numpy as np

    from paper_2110_10762_b200 import inputs
    cfg = base_config(problem={"name": "heat2d", "n": 12, "t_final": 0.02, "seed": 3},
                      fine={"rule": "forward-euler", "steps": 50, "dtype": "float32"},
                      coarse={"rule": "backward-euler", "steps": 1, "solver": "cg"},
                      device_runs=[{"seed": 4, "domains": 2, "delay_frac": 0.1}], analysis=False)
    c = parse_config(cfg)
    assert c.ivp.shape == (12, 12)
    assert np.array_equal(c.ivp.u0, inputs.sine_u0((12, 12), seed=3))
    assert c.fine.dtype == "float32" and c.coarse.dtype == "float64" and c.coarse.solver == "cg"
    assert c.device_runs[0].domains == 2 and not c.analysis
    path = tmp_path / "c.json"
    path.write_text(json.dumps(c.to_dict()), encoding="utf-8")
    c2 = load_config(path)
    assert c2.to_dict() == c.to_dict()
    h1 = parse_config(base_config(problem={"name": "heat1d", "n_interior": 64, "boundary_left": 0.0,
                                           "boundary_right": 0.0, "sine_modes": 8, "seed": 0}))
    assert np.array_equal(h1.ivp.u0, inputs.sine_u0_1d(64, 8, 0))


def _write_summary(path, rows):
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.DictWriter(fh, fieldnames=SUMMARY_COLUMNS)
        w.writeheader()
        for r in rows:
            w.writerow({k: r.get(k, "") for k in SUMMARY_COLUMNS})


def test_table_sorting_and_format(tmp_path):
    rows = [
        {"label": "x", "p": 8, "mode": "async-device", "policy": "device", "seed": 3, "iterations": 12,
         "model_cost": "300.0", "error_vs_oracle": "0.0"},
        {"label": "x", "p": 8, "mode": "async", "policy": "random-fair", "seed": 2, "delay_bound": 2,
         "iterations": 9, "model_cost": "250.5", "error_vs_oracle": "1.5e-9"},
        {"label": "x", "p": 4, "mode": "sync", "iterations": 3, "model_cost": "120.0", "fitted_overhead": "0.25",
         "error_vs_oracle": "2e-12"},
        {"label": "x", "p": 8, "mode": "sequential", "model_cost": "200.0", "error_vs_oracle": "0.0"},
    ]
    src, dst = tmp_path / "s.csv", tmp_path / "t.csv"
    _write_summary(src, rows)
    emit_table(src, dst)
    with open(dst, newline="", encoding="utf-8") as fh:
        out = list(csv.DictReader(fh))
    assert list(out[0].keys()) == TABLE_COLUMNS
    assert [(r["p"], r["mode"]) for r in out] == [("4", "sync"), ("8", "sequential"), ("8", "async"),
                                                  ("8", "async-device")]
    assert out[0]["fitted_overhead"] == "0.25" and out[1]["fitted_overhead"] == "-"
    assert out[2]["schedule"] == "random-fair/s2/D2" and out[3]["schedule"] == "device/s3"
    assert out[2]["error_vs_oracle"] == "1.50E-09" and out[1]["iterations"] == "-"


def test_table_rejects_foreign_csv(tmp_path, capsys):
    src = tmp_path / "s.csv"
    src.write_text("a,b\n1,2\n", encoding="utf-8")
    assert main(["table", "--in", str(src), "--out", str(tmp_path / "t.csv")]) == 1
