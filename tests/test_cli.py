"""The standalone CLI (paper_2205_00618_b200/cli.py) against the reference
CLI's interchange (cli.py:76-123): shapes.json + <slot>.bin data directories,
exit code 2 on input errors."""
import json
import os

import numpy as np
import pytest

import common
from paper_2205_00618_b200 import cli

SMALL = [c for c in common.index()["cases"] if c["size"] == "small"]
CASES = [c for c in SMALL if c["name"] in ("semiring_add_max", "conv_pad1_small", "mlp_bias_relu_small",
                                           "acc_maxpool", "acc_concat")]


def _graph_file(tmp_path, case):
    p = tmp_path / "g.json"
    p.write_text(common.graph_json(case["graph"]))
    return str(p)


def _write_dir(tmp_path, ins):
    d = tmp_path / "data"
    d.mkdir()
    for s, a in ins.items():
        np.ascontiguousarray(a, dtype="<f4").tofile(d / f"{s}.bin")
    (d / "shapes.json").write_text(json.dumps({str(s): list(a.shape) for s, a in ins.items()}))
    return str(d)


def test_compile_asm_and_json(tmp_path, capsys):
    case = CASES[0]
    g = _graph_file(tmp_path, case)
    assert cli.main(["compile", g]) == 0
    assert capsys.readouterr().out.startswith("launch.")
    assert cli.main(["compile", g, "--emit", "json"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["launches"] == len(out["steps"]) >= 1


@pytest.mark.parametrize("mutate,msg", [
    ("nofile", "no such file"), ("nomanifest", "missing"), ("badsize", "blob has"),
    ("badslot", "not used by the graph"), ("noblob", "missing blob"), ("noinput", "missing input slots"),
    ("badjson", "malformed"),
])
def test_run_input_errors_exit_2(tmp_path, capsys, mutate, msg):
    case = CASES[0]
    ins, _, _ = common.case_data(case)
    g = _graph_file(tmp_path, case)
    d = _write_dir(tmp_path, ins)
    if mutate == "nofile":
        g = str(tmp_path / "missing.json")
    elif mutate == "nomanifest":
        os.remove(os.path.join(d, "shapes.json"))
    elif mutate == "badsize":
        s = sorted(ins)[0]
        np.zeros(3, "<f4").tofile(os.path.join(d, f"{s}.bin"))
    elif mutate == "badslot":
        m = json.load(open(os.path.join(d, "shapes.json")))
        m["99"] = [1]
        json.dump(m, open(os.path.join(d, "shapes.json"), "w"))
    elif mutate == "noblob":
        os.remove(os.path.join(d, f"{sorted(ins)[0]}.bin"))
    elif mutate == "noinput":
        m = json.load(open(os.path.join(d, "shapes.json")))
        del m[str(sorted(ins)[0])]
        json.dump(m, open(os.path.join(d, "shapes.json"), "w"))
    elif mutate == "badjson":
        with open(g, "w") as f:
            f.write('{"vars": [], "nodes": [{"kind": "read"}]}')
    assert cli.main(["run", g, "--data", d]) == 2
    assert msg in capsys.readouterr().err


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_run_data_dir_matches_oracle(tmp_path, capsys, case):
    ins, ref, _ = common.case_data(case)
    g = _graph_file(tmp_path, case)
    d = _write_dir(tmp_path, ins)
    assert cli.main(["run", g, "--data", d]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["ok"] and out["counters"]["launches"] >= 1
    man = json.load(open(os.path.join(d, "shapes.json")))
    for slot, r in ref.items():
        assert str(slot) in man
        got = np.fromfile(os.path.join(d, f"{slot}.bin"), "<f4").reshape(man[str(slot)])
        ok, m = common.check_case(case["rule"], got, r, has_sigmoid=False)
        assert ok, f"{case['name']} slot {slot}: {m}"


@pytest.mark.gpu
def test_bench_payload(tmp_path, capsys):
    g = _graph_file(tmp_path, CASES[0])
    assert cli.main(["bench", g, "--min-ms", "5"]) == 0
    st = json.loads(capsys.readouterr().out)
    assert st["repeats"] >= 1 and st["gflops"] > 0 and st["flops"] > 0
