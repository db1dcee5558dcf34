"""CLI harness (cli.py mirror of the reference's cli.py:95-291): config handling and exit codes
on CPU; the commands themselves on the GPU."""

import json

import pytest

from paper_2007_07336_b200 import cli


def _args(cmd, **kw):
    ns = cli.build_parser().parse_args([cmd])
    for k, v in kw.items():
        setattr(ns, k, v)
    return ns


def test_defaults_and_flag_overrides():
    cfg = cli.load_config("converge", _args("converge", depths="16,32", tol=1e-8))
    assert cfg["depths"] == [16, 32] and cfg["tol"] == 1e-8 and cfg["width"] == 16


def test_unknown_config_key_exits_2(tmp_path, capsys):
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"depths": [8], "bogus": 1}))
    assert cli.main(["converge", "--config", str(p)]) == cli.EXIT_CONFIG
    assert "unknown keys" in capsys.readouterr().err


def test_flag_not_applying_exits_2():
    assert cli.main(["oracle-check", "--batches", "1,2"]) == cli.EXIT_CONFIG


def test_bad_int_list_exits_2():
    assert cli.main(["converge", "--depths", "8,x"]) == cli.EXIT_CONFIG


def test_workers_key_and_flag_like_the_reference(tmp_path):
    """reference configs carry "workers" (cli.py:42,55,83) and --workers exists."""
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"depths": [8], "workers": [2]}))
    cfg = cli.load_config("converge", _args("converge", config=str(p)))
    assert cfg["workers"] == [2]
    cfg = cli.load_config("scale", _args("scale", workers="1,2,4", gpus="1,2"))
    assert cfg["workers"] == [1, 2, 4] and cfg["gpus"] == [1, 2]
    assert cli.main(["converge", "--workers", "0"]) == cli.EXIT_CONFIG
    assert cli.main(["converge", "--gpus", "2"]) == cli.EXIT_CONFIG  # scale only


def test_csv_layout(capsys):
    cli.write_rows(None, ["a", "b"], [[1, 0.5]])
    out = capsys.readouterr().out.splitlines()
    assert out[0].startswith("# generated ") and out[1] == "a,b" and out[2] == "1,0.5"


@pytest.mark.gpu
def test_commands_on_gpu(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    out = tmp_path / "conv.csv"
    assert cli.main(["converge", "--depths", "16,64", "--out", str(out)]) == cli.EXIT_OK
    lines = out.read_text().splitlines()
    assert lines[1] == "depth,cycle,residual_l2" and len(lines) > 4
    assert cli.main(["oracle-check", "--depths", "16,64", "--seed", "0", "--out",
                     str(tmp_path / "o.csv")]) == cli.EXIT_OK
    s = tmp_path / "s.csv"
    assert cli.main(["scale", "--batches", "1,4", "--workers", "1,2", "--gpus", "1,2",
                     "--out", str(s)]) == cli.EXIT_OK
    lines = s.read_text().splitlines()
    assert lines[1] == ("workers,gpus,batch,wall_seconds,layer_samples_per_s,bound,roofline_frac,"
                        "shared,checksum")
    rows = [ln.split(",") for ln in lines[2:]]
    assert len(rows) == 6 and {r[1] for r in rows} == {"1", "2"}
    assert len({r[-1] for r in rows}) == 1  # bitwise across workers, batches and GPU counts
    assert all(0.0 < float(r[6]) <= 1.0 for r in rows)
