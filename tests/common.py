"""Helpers shared by the tests: golden-case loading, seeded config inputs,
parity rules.  Reads only files under tests/golden/ (never /root/reference)."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def index() -> dict:
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return json.load(f)


def graph_json(rel: str) -> str:
    with open(os.path.join(GOLDEN, rel)) as f:
        return f.read()


def case_data(case: dict):
    d = np.load(os.path.join(GOLDEN, case["data"]))
    ins = {int(k[3:]): d[k] for k in d.files if k.startswith("in_")}
    ref = {int(k[4:]): d[k] for k in d.files if k.startswith("ref_")}
    vm = {int(k[3:]): d[k] for k in d.files if k.startswith("vm_")}
    return ins, ref, vm


def config(name: str) -> dict:
    for c in index()["configs"]:
        if c["name"] == name:
            return c
    raise KeyError(name)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def config_inputs(name: str, bias_nonzero: bool = False):
    """Seeded inputs of SURVEY §8(d) (draw order as listed); slot -> array."""
    if name == "C1":
        rng = np.random.default_rng(0)
        return {0: rng.uniform(-1, 1, (256, 256)).astype(np.float32),
                1: rng.uniform(-1, 1, (256, 256)).astype(np.float32)}
    if name == "C2":
        rng = np.random.default_rng(1)
        return {0: rng.uniform(-10, 10, (1024, 1024)).astype(np.float32),
                1: rng.uniform(-10, 10, (1024, 1024)).astype(np.float32)}
    if name in ("C3", "C3g"):
        rng = np.random.default_rng(2)
        x = rng.uniform(-1, 1, (8, 64, 56, 56)).astype(np.float32)
        w = rng.normal(0.0, np.sqrt(2.0 / 576.0), (64, 64, 3, 3)).astype(np.float32)
        if name == "C3":
            x = np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1)))
        return {0: x, 1: w}
    if name in ("C4", "C4a"):
        rng = np.random.default_rng(3)
        X = rng.normal(0, 0.02, (4096, 1024)).astype(np.float32)
        W = rng.normal(0, 0.02, (1024, 4096)).astype(np.float32)
        b = rng.normal(0, 0.02, (4096,)).astype(np.float32) if bias_nonzero else np.zeros(4096, np.float32)
        if name == "C4":
            return {0: X, 1: W, 2: b}
        return {0: X, 1: W, 2: np.ascontiguousarray(np.broadcast_to(b, (4096, 4096)))}
    if name == "C5":
        rng = np.random.default_rng(4)
        A = rng.uniform(-1, 1, (16384, 16384)).astype(np.float32)
        B = rng.uniform(-1, 1, (16384, 16384)).astype(np.float32)
        return {0: A, 1: B}
    raise KeyError(name)


RTOL, ATOL = 1e-4, 1e-5


def strict_ok(got, ref):
    got = np.asarray(got, np.float64).reshape(ref.shape)
    same = np.isinf(ref) & (got == ref)
    return same | (np.abs(got - ref) <= ATOL + RTOL * np.abs(ref))


def ref_metric(got, ref) -> float:
    got = np.asarray(got, np.float64).reshape(ref.shape)
    fin = np.isfinite(ref)
    if not np.array_equal(got[~fin], ref[~fin]):
        return float("inf")
    if not fin.any():
        return 0.0
    return float(np.max(np.abs(got[fin] - ref[fin]) / np.maximum(np.abs(ref[fin]), 1.0)))


def value_exact(got, ref) -> bool:
    """got == float32(ref) elementwise (±0 compare equal, infs must match)."""
    want = np.asarray(ref, np.float64).astype(np.float32)
    got = np.asarray(got, np.float32).reshape(want.shape)
    return bool(np.array_equal(got, want))


def check_case(rule: str, got, ref, has_sigmoid=False) -> tuple[bool, str]:
    if rule == "bitexact" or (rule == "exact" and not has_sigmoid):
        ok = value_exact(got, ref)
        return ok, f"exact={ok} metric={ref_metric(got, ref):.2e}"
    m = ref_metric(got, ref)
    frac = float(strict_ok(got, ref).mean())
    return m <= 1e-4, f"metric={m:.2e} strict_pass={frac:.5f}"
