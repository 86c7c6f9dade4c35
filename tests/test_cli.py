"""CLI front end: the reference's commands, flags and exit codes
(cli.py:158-197, :397-420).  Argument handling runs on the CPU; the
synth -> train -> eval -> bench -> rerun round trip needs the GPU engine."""

import json
import os

import numpy as np
import pytest

from paper_1808_03843_b200 import cli


def test_usage_errors_exit_1(capsys):
    assert cli.main([]) == 1
    assert cli.main(["train"]) == 1  # --train is required
    assert cli.main(["bogus"]) == 1
    assert "usage error" in capsys.readouterr().err


def test_missing_files_exit_2(tmp_path, capsys):
    assert cli.main(["eval", "--model", str(tmp_path / "none.cmfm"), "--test", str(tmp_path / "t.tsv")]) == 2
    assert cli.main(["train", "--train", str(tmp_path / "none.tsv")]) == 2
    assert "data error" in capsys.readouterr().err


def test_bad_text_exit_2(tmp_path):
    p = tmp_path / "bad.tsv"
    p.write_text("0\t1\t2\n0\t1\n")
    assert cli.main(["train", "--train", str(p)]) == 2


def test_out_of_scope_engines_are_refused(tmp_path):
    p = tmp_path / "ok.tsv"
    p.write_text("0\t1\t2\n1\t0\t1\n")
    assert cli.main(["train", "--train", str(p), "--engine", "sgd"]) == 1
    assert cli.main(["bench", "--train", str(p), "--mode", "compare"]) == 1


def test_half_exact_is_a_usage_error():
    args = cli.build_parser().parse_args(["train", "--train", "x", "--solver", "exact", "--half"])
    with pytest.raises(cli.UsageError):
        cli._solver_config(args)
    cfg = cli._solver_config(cli.build_parser().parse_args(["train", "--train", "x", "--half"]))
    assert (cfg.method, cfg.precision, cfg.cg_iters) == ("cg", "fp16", 6)


def test_one_based_shift(tmp_path):
    p = tmp_path / "one.csv"
    p.write_text("1,1,5\n3,2,1\n")
    t, m, n = cli._load_triples(str(p), "csv", True)
    assert list(t.user) == [0, 2] and list(t.item) == [0, 1] and (m, n) == (3, 2)
    p.write_text("0,1,5\n")
    with pytest.raises(Exception, match="below 1"):
        cli._load_triples(str(p), "csv", True)


@pytest.mark.gpu
def test_cli_round_trip(tmp_path, capsys):
    pre = str(tmp_path / "syn")
    assert cli.main(["synth", "--m", "300", "--n", "200", "--f", "8", "--density", "0.1",
                     "--noise", "0.05", "--out", pre]) == 0
    for ext in (".tsv", ".cmfr", ".truth.cmfm", ".manifest.json"):
        assert os.path.exists(pre + ext)
    model, report = str(tmp_path / "m.cmfm"), str(tmp_path / "r.jsonl")
    assert cli.main(["train", "--train", pre + ".cmfr", "--test", pre + ".tsv", "--factors", "8",
                     "--epochs", "3", "--half", "--model-out", model, "--report-out", report]) == 0
    out = capsys.readouterr().out
    assert "epochs=3" in out and "rmse=" in out
    assert cli.main(["eval", "--model", model, "--test", pre + ".tsv", "--train", pre + ".tsv"]) == 0
    out = capsys.readouterr().out
    assert "rmse=" in out and "objective=" in out
    assert cli.main(["train", "--train", pre + ".tsv", "--engine", "implicit", "--factors", "8",
                     "--epochs", "2", "--model-out", model, "--report-out", report]) == 2  # negative ratings
    bench = str(tmp_path / "b")
    assert cli.main(["bench", "--train", pre + ".cmfr", "--test", pre + ".tsv", "--factors", "8",
                     "--epochs", "2", "--out", bench]) == 0
    rows = [json.loads(l) for l in open(bench + ".rows.jsonl")]
    assert [r["config"] for r in rows] == ["exact-fp32", "cg-fp32", "cg-fp16"]
    assert all(np.isfinite(r["final_rmse"]) for r in rows)
    assert cli.main(["rerun", bench + ".manifest.json"]) == 0
