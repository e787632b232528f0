"""Dataset loaders (datasets.hpp, cases of proj/tests/test_datasets.cpp) and the
host side of the `ihs` CLI (ihs_cli.cpp): argument and dataset errors, default
regularization paths, JSON layouts (serialize.hpp). CPU only."""
import json

import numpy as np
import pytest

from paper_2006_05874_b200 import cli, ihs
from paper_2006_05874_b200 import path as P
from paper_2006_05874_b200.datasets import Dataset, DatasetSource, load_csv, load_libsvm


def _file(tmp_path, name, content):
    f = tmp_path / name
    f.write_text(content)
    return str(f)


# ------------------------------------------------------------ load_csv (test_datasets.cpp:55-88)
def test_csv_well_formed(tmp_path):
    ds = load_csv(_file(tmp_path, "ok.csv", "1,2,5\n3,4,6\n"))
    assert (ds.n(), ds.d()) == (2, 2)
    assert ds.A.tolist() == [[1.0, 2.0], [3.0, 4.0]] and ds.b.tolist() == [5.0, 6.0]
    assert ds.source == DatasetSource.CSVFile and ds.provenance.startswith("csv:")


def test_csv_errors(tmp_path):
    with pytest.raises(ihs.ParseError):
        load_csv(_file(tmp_path, "empty.csv", ""))
    with pytest.raises(ihs.ParseError) as e:
        load_csv(_file(tmp_path, "bad.csv", "1,2,3\n4,x,6\n"))
    assert e.value.line == 2
    with pytest.raises(ihs.ShapeError):
        load_csv(_file(tmp_path, "ragged.csv", "1,2,3\n4,5\n"))
    with pytest.raises(ihs.InvalidInput):
        load_csv(str(tmp_path / "does_not_exist.csv"))
    with pytest.raises(ihs.ParseError, match="trailing"):
        load_csv(_file(tmp_path, "trail.csv", "1,2x,3\n"))
    with pytest.raises(ihs.ParseError, match="at least one feature"):
        load_csv(_file(tmp_path, "one.csv", "1\n"))
    with pytest.raises(ihs.InvalidInput, match="non-finite"):
        load_csv(_file(tmp_path, "inf.csv", "1,inf,3\n"))
    # blank lines are skipped but counted; whitespace around numbers as std::stod allows
    ds = load_csv(_file(tmp_path, "blank.csv", "\n 1, 2 ,3\n\n4,5,6 \n"))
    assert ds.A.tolist() == [[1.0, 2.0], [4.0, 5.0]]
    with pytest.raises(ihs.ParseError) as e:
        load_csv(_file(tmp_path, "bad2.csv", "\n1,2,3\n\n4,,6\n"))
    assert e.value.line == 4


# ------------------------------------------------------------ load_libsvm (test_datasets.cpp:90-123)
def test_libsvm_cases(tmp_path):
    ds = load_libsvm(_file(tmp_path, "ok.svm", "1 1:0.5 3:2\n"))
    assert (ds.n(), ds.d()) == (1, 3) and ds.A.tolist() == [[0.5, 0.0, 2.0]] and ds.b.tolist() == [1.0]
    ds = load_libsvm(_file(tmp_path, "two.svm", "-1 2:1\n0.5 4:3\n"))
    assert (ds.n(), ds.d()) == (2, 4) and ds.A[0, 1] == 1.0 and ds.A[1, 3] == 3.0 and ds.b[0] == -1.0
    with pytest.raises(ihs.ParseError):
        load_libsvm(_file(tmp_path, "zero.svm", "1 0:2\n"))
    with pytest.raises(ihs.ParseError):
        load_libsvm(_file(tmp_path, "pair.svm", "1 5\n"))
    with pytest.raises(ihs.ParseError):
        load_libsvm(_file(tmp_path, "empty.svm", "\n\n"))
    with pytest.raises(ihs.ParseError, match="no features"):
        load_libsvm(_file(tmp_path, "nofeat.svm", "1\n2\n"))
    with pytest.raises(ihs.ParseError, match="malformed feature index"):
        load_libsvm(_file(tmp_path, "idx.svm", "1 a:2\n"))
    with pytest.raises(ihs.InvalidInput):
        load_libsvm(str(tmp_path / "missing.svm"))


# ------------------------------------------------------------ CLI host logic
def test_cli_errors_exit_2(tmp_path, capsys):
    assert cli.main(["solve", "--nu", "1"]) == 2
    assert "no dataset given" in capsys.readouterr().err
    assert cli.main(["synth", "--csv", "x.csv"]) == 2
    assert "synth requires" in capsys.readouterr().err
    bad = _file(tmp_path, "bad.csv", "1,2\n3,q\n")
    assert cli.main(["path", "--csv", bad]) == 2
    assert "line 2" in capsys.readouterr().err
    ok = _file(tmp_path, "ok.csv", "1,2,5\n3,4,6\n")
    assert cli.main(["compare", "--csv", ok, "--solvers", "adaptive,nope"]) == 2
    assert "unknown solver 'nope'" in capsys.readouterr().err
    assert cli.main(["path", "--csv", ok, "--nus", "0.1,0.5"]) == 2
    assert "strictly decreasing" in capsys.readouterr().err
    assert cli.main(["compare", "--csv", ok, "--repeats", "0"]) == 2


def test_default_nus():  # ihs_cli.cpp:102-117
    real = Dataset(np.zeros((2, 1)), np.zeros(2), DatasetSource.CSVFile)
    syn = Dataset(np.zeros((2, 1)), np.zeros(2), DatasetSource.SyntheticExp)
    assert cli.parse_nus("", real) == [1e4, 1e3, 1e2, 1e1, 1.0, 0.1, 0.01]
    assert cli.parse_nus("", syn) == [1.0, 0.1, 0.01, 0.001, 0.0001]
    assert cli.parse_nus("1,0.5,0.25", real) == [1.0, 0.5, 0.25]


def test_json_layouts():  # serialize.hpp:26-117
    rep = ihs.SolveReport(x=np.array([1.0, 2.0]), iterations=3, final_m=8, converged=True)
    rep.log = [ihs.IterationRecord(1, 8, 0.5, 1.0, ihs.StepKind.Resketch)]
    j = cli.report_json(rep)
    assert set(j) == {"iterations", "rejected", "final_m", "r1", "r_final", "converged", "sketch_exhausted",
                      "wall_seconds", "recompute_r_after_resketch", "tuning", "counters", "log", "x"}
    assert j["log"][0]["branch"] == "resketch" and j["x"] == [1.0, 2.0] and j["counters"]["total"] == 0
    s = P.RunSummary(solver="cg", nu=0.5, x=np.array([1.0]), ok=False, error="boom")
    js = cli.summary_json(s)
    assert js["error"] == "boom" and "delta" not in js
    s.delta = 0.25
    assert cli.summary_json(s)["delta"] == 0.25
    pr = P.PathResult(nus=[1.0], entries=[s], cumulative_seconds=[0.1])
    assert set(cli.path_json(pr)) == {"nus", "cumulative_seconds", "entries"}
    cr = P.ComparisonReport(nus=[1.0], repeats=2, eps=1e-10, aggregates=[P.SolverAggregate(label="cg",
                                                                                          mean_cumulative=[0.2])])
    cj = json.loads(json.dumps(cli.comparison_json(cr)))
    assert cj["solvers"][0]["solver"] == "cg" and cj["solvers"][0]["mean_cumulative_seconds"] == [0.2]
