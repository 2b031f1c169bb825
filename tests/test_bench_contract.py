"""bench.py's reference arm runs on CPU (no GPU needed): its JSON line must
keep the driver contract (one line, metric/value/unit/impl/cpu_baseline/e2e)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                         text=True, timeout=600, cwd=ROOT, env=e)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0", "--ref-budget", "0.2"])
    assert d["impl"] == "reference" and d["unit"] == "GFLOP/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and "sample" in cb
    assert d["metric"].startswith("GFLOP/s, C1")


def test_reference_arm_nonzero_rank_is_silent():
    e = {"RANK": "1", "WORLD_SIZE": "2"}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "1", "--warmup", "0", "--ref-budget", "0.1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env={**os.environ, **e})
    assert out.returncode == 0 and out.stdout.strip() == ""
