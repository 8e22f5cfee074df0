"""CLI (reference cli.py and test_cli.py): usage errors exit 1, the device
flag, trace files in the blockeig-trace-v1 schema, plot from traces.  Runs that need a GPU
are marked gpu."""

import pytest

from paper_1407_7506_b200.cli import main, render_convergence_svg
from paper_1407_7506_b200.trace import TraceRecord, parse_trace_csv, trace_to_csv


def test_usage_errors_exit_1(capsys):
    assert main(["solve"]) == 1
    assert main(["solve", "--solver", "ppcg", "--problem", "lap1d:20", "--k", "0"]) == 1
    assert main(["solve", "--solver", "ppcg", "--problem", "nope:1", "--k", "2"]) == 1
    assert main(["solve", "--solver", "ppcg", "--problem", "lap1d:20", "--k", "2", "--device", "cpu"]) == 1
    assert main(["solve", "--solver", "ppcg", "--problem", "lap1d:20", "--k", "2", "--ngpus", "2"]) == 1
    assert main(["compare", "--solvers", "ppcg", "--problem", "lap1d:20", "--k", "2"]) == 1
    assert main(["solve", "--solver", "ppcg", "--problem", "lap1d:20", "--k", "2", "--rr-period", "x"]) == 1
    assert "error:" in capsys.readouterr().err


def test_plot_from_traces(tmp_path):
    recs = [TraceRecord(i, 1.0 / i, 10.0 ** -i, 0, 10 * i, float(i)) for i in range(1, 6)]
    p = tmp_path / "run.csv"
    p.write_text(trace_to_csv(recs))
    assert parse_trace_csv(p) == recs
    out = tmp_path / "plot.svg"
    assert main(["plot", str(p), "--out", str(out)]) == 0
    assert out.read_text().startswith("<svg") and "polyline" in out.read_text()
    assert "polyline" in render_convergence_svg([("a", [1, 2], [1e-1, 1e-3])])


@pytest.mark.gpu
def test_solve_and_compare_on_device(cuda, tmp_path, capsys):
    tr = tmp_path / "t.csv"
    rc = main(["solve", "--solver", "ppcg", "--problem", "lap1d:200", "--k", "4", "--tol", "1e-7",
               "--max-iter", "2000", "--trace-out", str(tr), "--json"])
    assert rc == 0
    assert "status: converged" in capsys.readouterr().out
    assert len(parse_trace_csv(tr)) > 0 and (tmp_path / "t.csv.json").exists()
    rc = main(["compare", "--solvers", "ppcg,lobpcg,davidson", "--problem", "rand:80,0.3", "--k", "4",
               "--tol", "1e-8", "--max-iter", "400", "--trace-out", str(tmp_path / "c_"),
               "--plot-out", str(tmp_path / "c.svg")])
    assert rc == 0
    for s in ("ppcg", "lobpcg", "davidson"):
        assert (tmp_path / f"c_{s}.csv").exists()
    rc = main(["solve", "--solver", "lobpcg", "--problem", "lap1d:100", "--k", "3", "--max-iter", "2"])
    assert rc == 2


@pytest.mark.gpu
def test_solve_matrix_market_problem_on_device(cuda, tmp_path, capsys):
    """`--problem mm:<path>` (reference cli.py problem grammar): the solve's reported eigenvalues
    are those of the file's matrix (dense eigvalsh), trace and JSON report written."""
    import json

    import numpy as np

    from paper_1407_7506_b200 import random_hermitian
    from paper_1407_7506_b200.mmio import write_matrix_market

    a = random_hermitian(120, 0.1, seed=77)
    mm = tmp_path / "a.mtx"
    write_matrix_market(a, mm)
    tr = tmp_path / "mm.csv"
    rc = main(["solve", "--solver", "ppcg", "--problem", f"mm:{mm}", "--k", "4", "--tol", "1e-9",
               "--max-iter", "500", "--trace-out", str(tr), "--json"])
    assert rc == 0
    out = capsys.readouterr().out
    assert "status: converged" in out
    vals = [float(ln) for ln in out.split("eigenvalues:")[1].split()]
    lam = np.linalg.eigvalsh(a.to_dense())[:4]
    assert np.allclose(vals, lam, rtol=1e-8, atol=1e-10)
    iters = int(out.split("iterations:")[1].split()[0])
    rows = parse_trace_csv(tr)
    assert rows and rows[-1].iteration == iters
    doc = json.loads((tmp_path / "mm.csv.json").read_text())
    assert doc["schema"] == "blockeig-trace-v1" and len(doc["records"]) == len(rows)
