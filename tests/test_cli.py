"""CLI contract (reference cli.py): exit codes and routing onto the engine."""

import json

import pytest

from paper_2605_14103_b200 import cli


def test_missing_case_is_input_error(capsys):
    assert cli.main(["solve", "--case", "/nonexistent/x.m"]) == 1
    assert "error: io" in capsys.readouterr().err


def test_bad_schema_is_input_error(tmp_path, capsys):
    p = tmp_path / "bad.json"
    p.write_text(json.dumps({"schema": "acpflow-zbus-network/1", "buses": []}))
    assert cli.main(["solve", "--case", str(p)]) == 1
    assert "error: schema" in capsys.readouterr().err


def test_unknown_kind_is_input_error(tmp_path):
    p = tmp_path / "x.txt"
    p.write_text("hello")
    assert cli.main(["solve", "--case", str(p)]) == 1


@pytest.mark.gpu
def test_solve_and_verify_on_gpu(tmp_path):
    out = tmp_path / "r.json"
    assert cli.main(["solve", "--case", "case118", "--batch", "16", "--seed", "1010",
                     "--out", str(out)]) == 0
    doc = json.loads(out.read_text())
    assert doc["report"]["aggregate"]["n_converged"] == 16
    assert len(doc["solutions"]) == 16
    assert cli.main(["verify", "--case", "case118"]) == 0
    assert cli.main(["verify", "--case", "ieee13"]) == 0
    csv = tmp_path / "b.csv"
    assert cli.main(["bench", "--case", "ieee13", "--batch", "64", "--out", str(csv)]) == 0
    assert csv.read_text().splitlines()[0].startswith("case,kind,batch_size")


@pytest.mark.gpu
def test_solve_with_gmres_step_on_gpu(tmp_path):
    # --step gmres --precond fd|none: the reference's own Newton step on the GPU
    for pre in ("fd", "none"):
        out = tmp_path / f"g_{pre}.json"
        assert cli.main(["solve", "--case", "case14", "--batch", "8", "--seed", "1010", "--step", "gmres",
                         "--precond", pre, "--out", str(out)]) == 0
        doc = json.loads(out.read_text())
        assert doc["report"]["aggregate"]["n_converged"] == 8


def test_step_option_validated():
    from paper_2605_14103_b200 import transmission as tm
    with pytest.raises(ValueError):
        tm.NewtonOptions(step="cg")
    with pytest.raises(SystemExit):
        cli.build_parser().parse_args(["solve", "--case", "case14", "--step", "cg"])


@pytest.mark.gpu
@pytest.mark.parametrize("case,batch", [("case118", 16), ("ieee13", 32)])
def test_solve_document_is_python_json(case, batch, tmp_path):
    """The natively written solve-result document (acpf_solve_result_json)
    re-serialises to the same bytes under the reference's json.dumps(indent=1)
    (cli.py:154): every float is repr-exact, the layout is json's."""
    out = tmp_path / "r.json"
    assert cli.main(["solve", "--case", case, "--batch", str(batch), "--seed", "1010", "--out", str(out)]) == 0
    text = out.read_text(encoding="utf-8")
    doc = json.loads(text)
    assert json.dumps(doc, indent=1) + "\n" == text
    assert doc["report"]["aggregate"]["count"] == batch
    csv = tmp_path / "r.csv"
    assert cli.main(["solve", "--case", case, "--batch", str(batch), "--seed", "1010", "--format", "csv",
                     "--out", str(csv)]) == 0
    rows = csv.read_text().splitlines()
    assert rows[0] == "index,converged,iterations,residual,error,wall_time" and len(rows) == batch + 1
