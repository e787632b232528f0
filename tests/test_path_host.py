"""Host logic of the regularization-path driver (bench.hpp): argument checks that
fire before any device work, solver names, aggregation and the plot CSV format.
CPU only."""
import io

import pytest

from paper_2006_05874_b200 import ihs, path as P


def test_path_argument_checks():  # test_bench.cpp:21-24, 131-133
    ds = P.Dataset(None, None)
    with pytest.raises(ihs.InvalidInput, match="strictly decreasing"):
        P.run_path(ds, [0.1, 0.5], P.SolverSpec(), 1e-10, 1)
    with pytest.raises(ihs.InvalidInput, match="strictly decreasing"):
        P.run_path(ds, [0.5, 0.5], P.SolverSpec(), 1e-10, 1)
    with pytest.raises(ihs.InvalidInput, match="empty"):
        P.run_path(ds, [], P.SolverSpec(), 1e-10, 1)
    with pytest.raises(ihs.InvalidInput, match="repeats"):
        P.compare_solvers(ds, [0.5], [P.SolverSpec()], 1e-10, 0, 1)
    with pytest.raises(ihs.InvalidInput, match="no solvers"):
        P.compare_solvers(ds, [0.5], [], 1e-10, 1, 1)


def test_solver_names():  # bench.hpp:19-27, 38-40
    assert [P.solver_name(i) for i in P.SolverId] == ["adaptive", "adaptive-gd", "cg", "pcg"]
    assert P.SolverSpec(id=P.SolverId.CG).name() == "cg"
    assert P.SolverSpec(id=P.SolverId.CG, label="mine").name() == "mine"
    s = P.SolverSpec()
    assert (s.rho, s.eta, s.m_initial, s.max_iters, s.enforce_validity) == (0.1, 0.01, 1, 2000, True)


def test_plot_csv_format():  # bench.hpp:244-254 (std::ostream default: 6 significant digits)
    rep = P.ComparisonReport(nus=[1.0, 0.1, 1e-5], repeats=1, eps=1e-10,
                             aggregates=[P.SolverAggregate(label="adaptive", mean_cumulative=[0.5, 1.25, 2.0]),
                                         P.SolverAggregate(label="cg", mean_cumulative=[1 / 3, 0.001234567, 3e7])])
    f = io.StringIO()
    P.write_plot_csv(f, rep)
    assert f.getvalue().splitlines() == ["nu,adaptive,cg", "1,0.5,0.333333", "0.1,1.25,0.00123457", "1e-05,2,3e+07"]
