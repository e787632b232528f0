"""The `ihs` CLI end to end on the device (ihs_cli.cpp subcommands solve / path /
compare / synth) and the synthetic spectra generator (test_datasets.cpp:24-53)."""
import json

import numpy as np
import pytest

from paper_2006_05874_b200 import cli, ihs
from paper_2006_05874_b200.datasets import SyntheticKind, generate_synthetic, load_csv

pytestmark = pytest.mark.gpu


def test_synthetic_spectra(gpu):
    ds = generate_synthetic(SyntheticKind.Exp, 12, 3, 1)
    np.testing.assert_allclose(np.linalg.svd(ds.A, compute_uv=False), [0.95, 0.9025, 0.857375], rtol=1e-10)
    ds = generate_synthetic(SyntheticKind.Poly, 16, 4, 2)
    np.testing.assert_allclose(np.linalg.svd(ds.A, compute_uv=False), [1.0, 0.5, 1 / 3, 0.25], rtol=1e-10)
    a, b = generate_synthetic(SyntheticKind.Exp, 20, 5, 77), generate_synthetic(SyntheticKind.Exp, 20, 5, 77)
    assert np.array_equal(a.A, b.A) and np.array_equal(a.b, b.b)
    assert np.linalg.norm(a.A - generate_synthetic(SyntheticKind.Exp, 20, 5, 78).A) > 0
    with pytest.raises(ihs.InvalidInput):
        generate_synthetic(SyntheticKind.Exp, 3, 5, 0)


def test_cli_solve_oracle_json(gpu, tmp_path, capsys):
    out = tmp_path / "r.json"
    rc = cli.main(["solve", "--synthetic", "exp", "--n", "512", "--d", "24", "--nu", "0.1", "--oracle",
                   "--out", str(out), "--sketch", "srht"])
    assert rc == 0
    j = json.loads(out.read_text())
    assert j["converged"] and j["delta"] <= 1e-6 and len(j["x"]) == 24 and j["nu"] == 0.1
    assert j["dataset"] == "synthetic-exp n=512 d=24 seed=0"
    assert any(e["branch"] == "resketch" for e in j["log"])
    assert "converged: yes" in capsys.readouterr().out


def test_cli_underdetermined_solve(gpu, O, tmp_path):
    rng = np.random.default_rng(3)
    # d = 200: the dual's Gaussian growth cap (d rows) leaves room to converge; at d = 40 the reference
    # itself stops with the sketch exhausted (exit status 1)
    A, b = rng.standard_normal((10, 200)), rng.standard_normal(10)
    f = tmp_path / "u.csv"
    f.write_text("".join(",".join(repr(float(v)) for v in list(A[i]) + [b[i]]) + "\n" for i in range(10)))
    assert cli.main(["solve", "--csv", str(f), "--nu", "0.5", "--out", str(tmp_path / "e.json"), "--sketch", "gaussian",
                     "--eps", "1e-10"]) == 0
    out = tmp_path / "u.json"
    assert cli.main(["solve", "--csv", str(f), "--nu", "0.5", "--oracle", "--out", str(out)]) == 0
    j = json.loads(out.read_text())
    # parity with the oracle's solve under the CLI's default config (the reference's stopping rule ends the
    # solve at r <= eps r_1, so x is compared with the oracle's x, and rel_error with the exact solution)
    x_or = O.solve_underdetermined(A, b, 0.5, O.default_config(max_iters=2000))[0]
    x = np.array(j["x"])
    assert np.linalg.norm(x - x_or) <= 1e-8 * (1 + np.linalg.norm(x_or))
    ref = A.T @ np.linalg.solve(A @ A.T + 0.25 * np.eye(10), b)
    assert j["rel_error"] == pytest.approx(np.linalg.norm(x - ref) / (1 + np.linalg.norm(ref)), rel=1e-6)


def test_cli_path_and_compare(gpu, tmp_path, capsys):
    f = tmp_path / "d.csv"
    assert cli.main(["synth", "--synthetic", "exp", "--n", "200", "--d", "12", "--data-seed", "4",
                     "--out", str(f)]) == 0
    ds = load_csv(str(f))
    g = generate_synthetic(SyntheticKind.Exp, 200, 12, 4)
    assert np.array_equal(ds.A, g.A) and np.array_equal(ds.b, g.b)  # repr round trip is exact
    out = tmp_path / "p.json"
    assert cli.main(["path", "--csv", str(f), "--nus", "1,0.1,0.01", "--solver", "pcg", "--rho", "0.5",
                     "--out", str(out), "--oracle"]) == 0
    j = json.loads(out.read_text())
    assert len(j["entries"]) == 3 and all(e["ok"] and e["delta"] <= 1e-6 for e in j["entries"])
    assert "nu          iters" in capsys.readouterr().out
    csv = tmp_path / "c.csv"
    assert cli.main(["compare", "--csv", str(f), "--nus", "1,0.1", "--solvers", "adaptive,cg", "--repeats", "2",
                     "--out", str(csv)]) == 0
    lines = csv.read_text().splitlines()
    assert lines[0] == "nu,adaptive,cg" and len(lines) == 3
    js = tmp_path / "c.json"
    assert cli.main(["compare", "--csv", str(f), "--nus", "0.5", "--solvers", "adaptive-gd,pcg", "--repeats", "1",
                     "--out", str(js)]) == 0
    assert [s["solver"] for s in json.loads(js.read_text())["solvers"]] == ["adaptive-gd", "pcg"]
