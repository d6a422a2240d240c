"""bench.py's driver contract on CPU: --gpus N launches N ranks (torchrun,
one process per GPU; shown here by the gloo dry run), fails loudly when
fewer devices are visible, and the reference arm times exactly the samples
it reports."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=300):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT)


def _json_line(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def test_gpus_n_launches_n_ranks():
    r = _run("--gpus", "3", "--dry-run")
    assert r.returncode == 0, r.stderr[-2000:]
    d = _json_line(r.stdout)
    assert d["n_gpus"] == 3 and len({x["pid"] for x in d["ranks"]}) == 3
    assert [x["rank"] for x in d["ranks"]] == [0, 1, 2]
    assert d["async_c4_partition"] == [[1, 21], [22, 42], [43, 64]]


def test_gpus_n_without_devices_fails_loudly():
    import torch
    if torch.cuda.device_count() >= 2:
        return
    r = _run("--gpus", "2")
    assert r.returncode == 2
    assert "CUDA device" in r.stderr


def test_reference_arm_times_what_it_reports():
    r = _run("--impl", "reference", "--steps", "2", "--warmup", "1", timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _json_line(r.stdout)
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1
    assert d["ms_per_step"] > 0 and d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] == os.cpu_count()
