"""Report formats and CLI of the step after the path (
gapsafe/bench.py:25-148, gapsafe/cli.py; schema tests modelled on
pkg/tests/test_bench_cli.py:27-76)."""

import csv
import json

import numpy as np
import pytest

from paper_1505_03410_b200 import report
from paper_1505_03410_b200.cli import build_parser, config_from_args


def _write_npz(path, X, y):
    np.savez(path, X=X, y=y)


def _data(n=25, p=40, seed=11):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, p)) * (rng.random((n, p)) < 0.6)
    y = X[:, :3] @ np.array([1.0, -2.0, 0.5]) + 0.1 * rng.standard_normal(n)
    return X, y


class TestRunConfig:
    def test_empty_rules_rejected(self):
        with pytest.raises(ValueError):
            report.RunConfig(rules=[], epsilons=[1e-4])

    def test_bad_rule_rejected(self):
        with pytest.raises(ValueError):
            report.RunConfig(rules=["banana"], epsilons=[1e-4])

    def test_bad_epsilon_rejected(self):
        with pytest.raises(ValueError):
            report.RunConfig(rules=["none"], epsilons=[])
        with pytest.raises(ValueError):
            report.RunConfig(rules=["none"], epsilons=[-1e-4])


def test_cli_parses_reference_arguments(tmp_path):
    args = build_parser().parse_args(["bench", "--data", "x.npz", "--rules", "none, gap_dome",
                                      "--eps", "1e-4,1e-6", "--grid-T", "7", "--out", str(tmp_path)])
    cfg = config_from_args(args)
    assert [r.value for r in cfg.rules] == ["none", "gap_dome"]
    assert cfg.epsilons == [1e-4, 1e-6] and cfg.grid_T == 7 and cfg.grid_delta == 3.0


@pytest.mark.gpu
def test_reports_match_reference_schemas(tmp_path):
    jsonschema = pytest.importorskip("jsonschema")
    import paper_1505_03410_b200 as gs
    X, y = _data()
    out = tmp_path / "out"
    cfg = report.RunConfig(rules=["none", "gap_sphere", "gap_dome"], epsilons=[1e-4], grid_T=5, grid_delta=2.0,
                           out_dir=str(out), seed=11)
    report.run_benchmark(cfg, gs.DesignMatrix(np.asfortranarray(X)), y)
    summary = json.loads((out / "summary.json").read_text())
    metadata = json.loads((out / "metadata.json").read_text())
    jsonschema.validate(summary, report.SUMMARY_SCHEMA)
    jsonschema.validate(metadata, report.METADATA_SCHEMA)
    assert metadata["seed"] == 11 and len(summary["runs"]) == 3
    for run in summary["runs"]:
        assert run["n_converged"] == run["n_lambdas"] == 5
    with open(out / "trace.csv", newline="") as fh:
        rows = list(csv.DictReader(fh))
    assert rows and list(rows[0].keys()) == report.TRACE_COLUMNS
    by_key = {}
    for r in rows:
        by_key.setdefault((r["rule"], r["t"]), []).append(int(r["n_active"]))
    for sizes in by_key.values():
        assert all(b <= a for a, b in zip(sizes, sizes[1:]))
    for name in ("trace.csv", "summary.json", "metadata.json"):
        assert b"\r" not in (out / name).read_bytes()


@pytest.mark.gpu
def test_cli_bench_end_to_end(tmp_path, capsys):
    from paper_1505_03410_b200.cli import main
    X, y = _data()
    path = tmp_path / "d.npz"
    _write_npz(path, X, y)
    assert main(["bench", "--data", str(path), "--rules", "none,gap_sphere,static", "--grid-T", "4",
                 "--out", str(tmp_path / "o")]) == 0
    assert "converged=4/4" in capsys.readouterr().out
