"""MatrixMarket input (reference problems.py:92-188 and its
test_problems.py::TestMatrixMarket cases): format checks, mirroring, duplicate summation,
error line numbers, bit-exact round trips."""

import numpy as np
import pytest

from paper_1407_7506_b200 import random_hermitian
from paper_1407_7506_b200.errors import ParseError, UnsupportedFormatError
from paper_1407_7506_b200.mmio import read_matrix_market, write_matrix_market

HDR_R = "%%MatrixMarket matrix coordinate real symmetric\n"
HDR_Z = "%%MatrixMarket matrix coordinate complex hermitian\n"


def _read(tmp_path, text):
    p = tmp_path / "m.mtx"
    p.write_text(text)
    return read_matrix_market(p)


def test_entries_mirrored_summed_and_comments(tmp_path):
    assert np.array_equal(_read(tmp_path, HDR_R + "2 2 1\n1 1 2.0\n").to_dense(), [[2.0, 0.0], [0.0, 0.0]])
    assert np.array_equal(_read(tmp_path, HDR_R + "2 2 1\n2 1 3.0\n").to_dense(), [[0.0, 3.0], [3.0, 0.0]])
    assert _read(tmp_path, HDR_R + "2 2 2\n2 1 3.0\n2 1 1.5\n").to_dense()[0, 1] == 4.5
    a = _read(tmp_path, HDR_R + "% c\n\n3 3 1\n% again\n3 1 -1.0\n")
    assert a.n == 3 and a.to_dense()[0, 2] == -1.0
    z = _read(tmp_path, HDR_Z + "2 2 2\n1 1 1.0 0.0\n2 1 0.5 -0.25\n").to_dense()
    assert z[1, 0] == 0.5 - 0.25j and z[0, 1] == 0.5 + 0.25j


@pytest.mark.parametrize("text", [
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 2.0\n",
    "%%MatrixMarket matrix coordinate pattern symmetric\n2 2 1\n1 1\n",
    "%%MatrixMarket matrix array real symmetric\n2 2\n1.0\n",
    "%%MatrixMarket matrix coordinate complex symmetric\n2 2 1\n1 1 1.0 0.0\n",
    HDR_R + "2 3 1\n1 1 1.0\n",
])
def test_unsupported_formats(tmp_path, text):
    with pytest.raises(UnsupportedFormatError):
        _read(tmp_path, text)


@pytest.mark.parametrize("text,line", [
    ("not a matrix market file\n", 1),
    (HDR_R + "2 2 2\n1 1 2.0\n2 oops 3.0\n", 4),
    (HDR_R + "2 2 1\n3 1 1.0\n", 3),
    (HDR_R + "2 2\n1 1 1.0\n", 2),
    (HDR_R + "2 2 1\n1 1 1.0 7\n", 3),
    (HDR_Z + "2 2 1\n1 1 1.0 0.5\n", 3),
    (HDR_R + "2 2 2\n1 1 1.0\n", 3),
])
def test_parse_errors_report_the_line(tmp_path, text, line):
    with pytest.raises(ParseError) as exc:
        _read(tmp_path, text)
    assert exc.value.line == line


def test_empty_file(tmp_path):
    with pytest.raises(ParseError):
        _read(tmp_path, "")


@pytest.mark.parametrize("cplx", [False, True])
def test_round_trip_bit_exact(tmp_path, cplx):
    a = random_hermitian(40, 0.3, seed=99, complex_field=cplx)
    p = tmp_path / "rt.mtx"
    write_matrix_market(a, p)
    b = read_matrix_market(p)
    assert b.n == a.n and b.symmetry == a.symmetry
    assert np.array_equal(a.to_dense(), b.to_dense())


@pytest.mark.gpu
@pytest.mark.parametrize("cplx", [False, True])
def test_matrix_market_operator_solves_like_the_oracle(cuda, tmp_path, cplx):
    """SURVEY §8(f) rank 3 end to end: an operator written to and read back from a MatrixMarket
    file (reference problems.py:92-188) is solved on the device exactly as the in-memory one,
    and like the CPU oracle on the parsed matrix."""
    from oracle import ppcg_oracle as O
    from paper_1407_7506_b200 import SolverOptions, ppcg_solve
    from util import HostCsr

    a = random_hermitian(160, 0.08, seed=31, complex_field=cplx)
    p = tmp_path / "op.mtx"
    write_matrix_market(a, p)
    b = read_matrix_market(p)
    opts = SolverOptions(k=5, sbsize=2, tol=1e-9, seed=4, max_iter=300)
    rb = ppcg_solve(b, opts=opts)
    ra = ppcg_solve(a, opts=opts)
    ref = O.oracle_solve(HostCsr(b._csr), None, opts=opts)
    assert rb.status == ra.status == ref.status == "converged"
    assert rb.iterations == ra.iterations and np.array_equal(rb.values, ra.values)  # same CSR, same run
    assert abs(rb.iterations - ref.iterations) <= 1
    assert np.allclose(rb.values, ref.values, rtol=1e-10, atol=1e-12)
