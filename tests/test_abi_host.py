"""CPU tests of the boundary and host logic: the C-ABI library loads and exports every
symbol include/ppcg_b200.h declares (no compute calls), the binding table matches, the
product fails loudly without a GPU, and the host-side pieces of the reference interface
(options, partition, locking, initial block, trace schema) behave like the reference."""

import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "ppcg_b200.h")
LIB = os.path.join(ROOT, "paper_1407_7506_b200", "libppcg_b200.so")


def declared_symbols():
    text = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|double|unsigned long long)\s+(bk_\w+)\s*\(", text, re.M)))


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built (run make)")
def test_library_exports_every_declared_symbol():
    import ctypes

    lib = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_table_covers_header():
    from paper_1407_7506_b200 import _lib

    assert sorted(_lib.EXPORTED) == declared_symbols()


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1407_7506_b200 import DeviceError, SolverOptions, laplacian_1d, ppcg_solve

    with pytest.raises(DeviceError):
        ppcg_solve(laplacian_1d(50), opts=SolverOptions(k=2, max_iter=3))


def test_options_validation_matches_reference():
    from paper_1407_7506_b200 import SolverOptions

    for bad in (dict(k=0), dict(k=2, sbsize=0), dict(k=2, tol=0.0), dict(k=2, rr_period=0),
                dict(k=2, orth_policy="sometimes"), dict(k=2, orth_scheme="qr"), dict(k=2, max_iter=-1),
                dict(k=2, nbuf=-1), dict(k=2, trace_tol=0.0), dict(k=2, orth_period=0)):
        with pytest.raises(ValueError):
            SolverOptions(**bad).validate()
    assert SolverOptions(k=64).resolved_nbuf() == 2
    assert SolverOptions(k=512).resolved_nbuf() == 11
    SolverOptions(k=3, rr_period=math.inf).validate()


def test_split_blocks_and_lock_count():
    from paper_1407_7506_b200.ppcg import lock_count, split_blocks

    assert split_blocks(10, 5) == [(0, 5), (5, 10)]
    assert split_blocks(7, 5) == [(0, 5), (5, 7)]
    assert split_blocks(0, 5) == []
    with pytest.raises(ValueError):
        split_blocks(-1, 5)
    with pytest.raises(ValueError):
        split_blocks(4, 0)
    assert split_blocks(523, 32)[-1] == (512, 523)
    # prefix-closed locking (rayleigh_ritz.py:95-108)
    assert lock_count([1.0, 2.0, 3.0], [1e-9, 1e-3, 1e-9], 1e-6) == 1
    assert lock_count([100.0, 2.0], [1e-5, 1e-9], 1e-6) == 2  # scaled by max(|theta|, 1)
    assert lock_count([0.5], [2e-6], 1e-6) == 0


def test_initial_block_draw_matches_reference_recipe():
    from paper_1407_7506_b200.errors import DimensionError
    from paper_1407_7506_b200.ppcg import draw_initial_block

    x = draw_initial_block(20, 4, False, 7)
    assert np.array_equal(x, np.random.default_rng(7).standard_normal((20, 4)))
    z = draw_initial_block(10, 3, True, 2)
    g = np.random.default_rng(2)
    ref = g.standard_normal((10, 3)) + 1j * g.standard_normal((10, 3))
    assert np.array_equal(z, ref)
    x0 = np.ones((20, 2))
    xp = draw_initial_block(20, 4, False, 7, x0)
    assert np.array_equal(xp[:, :2], x0)
    assert np.array_equal(xp[:, 2:], np.random.default_rng(7).standard_normal((20, 2)))
    with pytest.raises(DimensionError):
        draw_initial_block(20, 2, False, 0, np.ones((20, 3)))
    with pytest.raises(DimensionError):
        draw_initial_block(20, 2, False, 0, np.ones((19, 2)))


def test_trace_schema_roundtrip(tmp_path):
    from paper_1407_7506_b200.errors import ParseError
    from paper_1407_7506_b200.trace import TraceRecord, parse_trace_csv, trace_to_csv

    recs = [TraceRecord(1, 1.0 / 3.0, 0.123456789012345, 0, 66, 1.5), TraceRecord(2, -2.5, 1e-7, 3, 200, 2.0)]
    p = tmp_path / "t.csv"
    p.write_text(trace_to_csv(recs))
    back = parse_trace_csv(p)
    assert back == recs
    p.write_text("bad\n")
    with pytest.raises(ParseError):
        parse_trace_csv(p)


def test_config_generators_shapes():
    from paper_1407_7506_b200.problems import config_problem

    a, k, q, tol = config_problem(1)
    assert a.n == 4096 and a.nnz == 20224 and (k, q) == (64, 8)
    a, k, q, tol = config_problem(4, N=16)
    assert a.nnz == (3 * 16 - 2) ** 3
    c = a._csr
    assert abs(c - c.T).max() == 0
    a, k, q, tol = config_problem(5, N=16)
    assert a.nnz == 7 * 16 ** 3 - 6 * 16 ** 2
    c = a._csr
    assert abs(c - c.conj().T).max() == 0


def test_oracle_is_not_imported_by_the_product():
    import subprocess
    import sys

    code = ("import sys; import paper_1407_7506_b200 as p; import paper_1407_7506_b200.ppcg, "
            "paper_1407_7506_b200.kernels, paper_1407_7506_b200.operators; "
            "print(any(m.startswith('oracle') for m in sys.modules))")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.stdout.strip() == "False", out.stderr


def test_parallel_host_normals_bit_identical():
    """X0 draw (ppcg.py:414-438): the multi-threaded PCG64 draw equals numpy's sequential one."""
    from paper_1407_7506_b200.hostrng import standard_normal

    for seed, count, th in [(0, 3_000_000, 4), (7, 2_200_001, 3), (11, 4_500_000, 8), (2, 1000, 4)]:
        assert np.array_equal(standard_normal(seed, count, th), np.random.default_rng(seed).standard_normal(count))


def test_initial_block_matches_reference_draw():
    from paper_1407_7506_b200.ppcg import draw_initial_block

    for cplx in (False, True):
        n, kt = 20000, 120
        x = draw_initial_block(n, kt, cplx, 3)
        rng = np.random.default_rng(3)
        ref = rng.standard_normal((n, kt))
        if cplx:
            ref = ref + 1j * rng.standard_normal((n, kt))
        assert np.array_equal(x, ref)


def test_initial_block_source_rows_match_draw():
    """The unassembled X0 draw (hostrng.FlatDraw) hands out exactly the rows of the draw."""
    from paper_1407_7506_b200.ppcg import draw_initial_block, initial_block_source

    n, kt = 30000, 110
    ref = draw_initial_block(n, kt, False, 5)
    for lo, hi in ((0, n), (1234, 20001)):
        src = initial_block_source(n, kt, False, 5, None, lo, hi)
        out = np.empty((hi - lo, kt))
        for r0 in range(0, hi - lo, 7001):
            r1 = min(hi - lo, r0 + 7001)
            src.fill_rows(r0, r1, out[r0:r1])
        assert np.array_equal(out, ref[lo:hi])
    src = initial_block_source(n, kt, True, 5, None, 10, 20)
    assert np.array_equal(src, draw_initial_block(n, kt, True, 5)[10:20])
