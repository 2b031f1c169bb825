"""bench.py's reference arm runs on CPU (no GPU needed): its JSON line must
keep the driver contract (one line, metric/value/unit/impl/cpu_baseline/e2e)."""
import json
import os
import subprocess
import sys

import pytest

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
                          "--gpus", "2", "--steps", "1", "--warmup", "0", "--ref-budget", "0.1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env={**os.environ, **e})
    assert out.returncode == 0 and out.stdout.strip() == ""


def _clean_env():
    return {k: v for k, v in os.environ.items()
            if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}


def test_launcher_spawns_ranks_one_json_line():
    """--gpus 2 without WORLD_SIZE: bench.py re-runs itself as 2 ranks under
    torch.distributed.run; rank 0 alone prints, n_gpus is 2."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--config", "C1", "--steps", "1", "--warmup", "0", "--ref-budget", "0.1", "--no-vm"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=_clean_env())
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"


def test_world_size_must_match_gpus():
    e = {**_clean_env(), "RANK": "0", "WORLD_SIZE": "2", "LOCAL_RANK": "0"}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "4",
                          "--config", "C1", "--steps", "1", "--no-vm"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=e)
    assert out.returncode == 2 and "WORLD_SIZE" in out.stderr


@pytest.mark.gpu
def test_bench_c5_through_launcher():
    """The headline config through the torchrun launcher path (1 rank): one
    JSON line, n_gpus 1, the shard's sampled rows pass the f64 check."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--launch",
                          "--config", "C5", "--steps", "3", "--warmup", "3", "--no-per-config", "--no-cpu"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=_clean_env())
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["parity"]["ok"] and d["parity"]["ref_metric"] <= 1e-4, d["parity"]
    assert d["clocks"]["sm_mhz"], d["clocks"]


@pytest.mark.gpu
def test_bench_gather_timer_single_rank():
    """The optional C-shard all-gather timer of N>1 runs (bench.time_gather)
    on a one-rank NCCL group: the code path the 2/4/8-GPU lines take."""
    code = ("import os, torch, torch.distributed as dist, bench\n"
            "torch.cuda.set_device(0)\n"
            "dist.init_process_group('nccl', device_id=torch.device('cuda', 0))\n"
            "g = bench.time_gather(torch, 1, 1024, 4096)\n"
            "assert g['ms'] > 0 and g['bytes_received_per_rank'] == 0, g\n"
            "from paper_2205_00618_b200 import shard\n"
            "comm = shard.nccl_comm()\n"
            "x = torch.arange(12, dtype=torch.float32, device='cuda').reshape(3, 4)\n"
            "y = torch.empty_like(x)\n"
            "shard.gather_rows_native(comm, x, y, torch.cuda.current_stream().cuda_stream)\n"
            "torch.cuda.synchronize()\n"
            "assert torch.equal(x, y)\n"
            "comm.close()\n"
            "dist.destroy_process_group()\n"
            "print('ok')\n")
    env = {**os.environ, "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": "29517", "RANK": "0", "WORLD_SIZE": "1",
           "LOCAL_RANK": "0"}
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env=env)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
