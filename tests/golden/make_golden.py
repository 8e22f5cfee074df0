"""Generate golden vectors from the REFERENCE implementation (blockeig, /root/reference).

Run in the build container only (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py            # kernels, generators, config-1, small solves
    python tests/golden/make_golden.py --cfg2     # + config-2 first iterations (~3 min, 12 GB)
    python tests/golden/make_golden.py --cfg2-full  # config-2 solve to convergence (~40 min, 12 GB)
    python tests/golden/make_golden.py --scaled     # configs 3-5 on scaled grids, q = 64

Every fixture records the inputs (or their seeds/recipes) and the reference outputs.  The
CPU tests pin the oracle (oracle/ppcg_oracle.py) against these files; the GPU tests check
the device path against them.
"""

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import importlib  # noqa: E402

import blockeig as B  # noqa: E402  (reference, read-only)

BC = importlib.import_module("blockeig.core")
BP = importlib.import_module("blockeig.ppcg")
BR = importlib.import_module("blockeig.rayleigh_ritz")

from paper_1407_7506_b200 import problems as P  # noqa: E402  (our generators, pure host code)


def g(n, m, seed, cplx=False):
    r = np.random.default_rng(seed)
    x = r.standard_normal((n, m))
    if cplx:
        x = x + 1j * r.standard_normal((n, m))
    return x


def kernels():
    out = {}
    # block_inner (core.py:43-49)
    x, y = g(50, 7, 1), g(50, 5, 2)
    out["gram_x"], out["gram_y"], out["gram_out"] = x, y, BC.block_inner(x, y)
    xz, yz = g(40, 4, 3, True), g(40, 6, 4, True)
    out["gramz_x"], out["gramz_y"], out["gramz_out"] = xz, yz, BC.block_inner(xz, yz)
    # solve_pencil (core.py:175-202), real d=24 want=8 and d=96 want=32, complex d=12 want=5
    for tag, d, want, cplx, seed in (("p24", 24, 8, False, 5), ("p96", 96, 32, False, 6), ("pz12", 12, 5, True, 7)):
        a = g(d, d, seed, cplx)
        a = 0.5 * (a + a.conj().T)
        gg = g(d, d + 3, seed + 100, cplx)
        b = gg @ gg.conj().T + 0.1 * np.eye(d)
        sol = BC.solve_pencil(BC.SmallPencil(a, b), want)
        out[f"{tag}_a"], out[f"{tag}_b"], out[f"{tag}_omega"], out[f"{tag}_c"] = a, b, sol.omega, sol.c
    # cholesky_qr (core.py:86-100) and the rank-deficiency column
    x = g(60, 6, 8)
    q, r = BC.cholesky_qr(x)
    out["cqr_x"], out["cqr_q"], out["cqr_r"] = x, q, r
    xd = x.copy()
    xd[:, 2] = xd[:, 0] + xd[:, 1]
    try:
        BC.cholesky_qr(xd)
        col = -1
    except B.RankDeficiencyError as e:
        col = e.column
    out["cqr_xd"], out["cqr_fail_col"] = xd, np.array(col)
    # polar_correction (core.py:106-124)
    xq = np.linalg.qr(g(30, 5, 9))[0] + 1e-3 * g(30, 5, 10)
    gram = xq.T @ xq
    out["polar_gram"], out["polar_poly"] = gram, BC.polar_correction(gram, 4)
    # convergence_metrics (rayleigh_ritz.py:71-92)
    xm = np.linalg.qr(g(80, 6, 11))[0]
    am = g(80, 80, 12)
    am = 0.5 * (am + am.T)
    m = BR.convergence_metrics(xm, am @ xm, prev_trace=1.5)
    out["met_x"], out["met_ax"] = xm, am @ xm
    out["met_out"] = np.array([m.rel_subspace_residual, m.trace_value, m.rel_trace_change])
    # block_update (ppcg.py:278-378) with P, q=4, and the engineered fallback
    n, q = 60, 4
    a = g(n, n, 13)
    a = 0.5 * (a + a.T)
    x = np.linalg.qr(g(n, q, 14))[0]
    w = g(n, q, 15)
    w -= x @ (x.T @ w)
    p = 1e-2 * g(n, q, 16)
    p -= x @ (x.T @ p)
    res = BP.block_update(x, w, p, ax=a @ x, aw=a @ w, ap=a @ p)
    out.update({"bu_a": a, "bu_x": x, "bu_w": w, "bu_p": p, "bu_xo": res.x, "bu_po": res.p, "bu_theta": res.theta,
                "bu_cx": res.c_x, "bu_cw": res.c_w, "bu_cp": res.c_p, "bu_cs": np.array(res.coeff_scale),
                "bu_fb": np.array(int(res.used_fallback))})
    d2 = np.diag([1.0, 2.0])
    res = BP.block_update(np.eye(2)[:, 1:2], np.eye(2)[:, 0:1], ax=d2 @ np.eye(2)[:, 1:2], aw=d2 @ np.eye(2)[:, 0:1])
    out["fb_x"], out["fb_theta"], out["fb_used"] = res.x, res.theta, np.array(int(res.used_fallback))
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)


def generators():
    """Pin our host-side mirrors of the reference generators (problems.py:191-286)."""
    out = {}
    cases = {
        "lap3d": (B.laplacian_3d(5, 4, 3), P.laplacian_3d(5, 4, 3)),
        "well": (B.well_problem(6, 6, 6, depth=40.0, seed=3), P.well_problem(6, 6, 6, depth=40.0, seed=3)),
        "rand": (B.random_hermitian(40, 0.3, seed=5), P.random_hermitian(40, 0.3, seed=5)),
        "randz": (B.random_hermitian(30, 0.4, seed=6, complex_field=True),
                  P.random_hermitian(30, 0.4, seed=6, complex_field=True)),
    }
    for k, (ref, _) in cases.items():
        c = ref._csr
        out[f"{k}_indptr"], out[f"{k}_indices"], out[f"{k}_data"] = c.indptr, c.indices, c.data
    ref_t = B.jacobi_preconditioner(cases["well"][0], shift=-90.0)
    out["well_jacobi"] = ref_t.d
    np.savez_compressed(os.path.join(HERE, "generators.npz"), **out)


def _report_arrays(prefix, rep, out, vectors=True):
    out[f"{prefix}_values"] = rep.values
    if vectors:
        out[f"{prefix}_vectors"] = rep.vectors
    tr = rep.trace
    out[f"{prefix}_trace"] = np.array([[r.iteration, r.trace_value, r.rel_resid, r.n_locked, r.n_matvec] for r in tr]).reshape(-1, 5)
    out[f"{prefix}_meta"] = np.array([rep.iterations, rep.matvecs, rep.rr_count, rep.breakdown_recoveries,
                                      1 if rep.status == "converged" else 0])
    out[f"{prefix}_final_rn"] = np.array(rep.diagnostics["final_residual_norms"])
    out[f"{prefix}_orth_loss"] = np.array(rep.diagnostics["orth_loss"])
    out[f"{prefix}_proj_defect"] = np.array(rep.diagnostics["proj_defect"])
    if rep.values_history:
        out[f"{prefix}_vhist"] = np.array(rep.values_history)


def solves():
    out = {}
    # BASELINE config 1: our generator's CSR fed to the reference's SparseHermitian
    ours, k, q, tol = P.config_problem(1)
    a = B.SparseHermitian(ours._csr, "symmetric")
    t = B.jacobi_preconditioner(a)
    t0 = time.time()
    rep = B.ppcg_solve(a, t, opts=B.SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=2000))
    print(f"config 1: {rep.status} {rep.iterations} it {rep.rr_count} RR {rep.matvecs} mv in {time.time() - t0:.1f}s")
    c1 = {}
    _report_arrays("cfg1", rep, c1)
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **c1)
    # reference-test problems (test_ppcg.py, test_acceptance.py)
    runs = {
        "lap1d": (B.laplacian_1d(500), None, dict(k=10, tol=1e-6, seed=0, max_iter=2000)),
        "rand90": (B.random_hermitian(90, 0.25, seed=17), None, dict(k=6, sbsize=2, tol=1e-9, seed=9, max_iter=80)),
        "randz60": (B.random_hermitian(60, 0.5, seed=4, complex_field=True), None,
                    dict(k=4, tol=1e-9, seed=1, max_iter=400)),
    }
    wa = B.well_problem(8, 8, 8, depth=80.0, seed=3)
    runs["well_tol4"] = (wa, B.jacobi_preconditioner(wa, shift=-90.0),
                         dict(k=10, nbuf=2, sbsize=5, rr_period=5, tol=1e-4, seed=1, max_iter=140))
    runs["well_tol6"] = (wa, B.jacobi_preconditioner(wa, shift=-90.0),
                         dict(k=10, nbuf=2, sbsize=5, rr_period=5, tol=1e-6, seed=1, max_iter=210))
    # scaled-down config 4 / config 5 structures (16^3 / 8^3)
    o4, _, _, _ = P.config_problem(4, N=12)
    a4 = B.SparseHermitian(o4._csr, "symmetric")
    runs["cfg4_n12"] = (a4, B.jacobi_preconditioner(a4), dict(k=32, sbsize=8, tol=1e-5, seed=0, max_iter=400))
    o5, _, _, _ = P.config_problem(5, N=8)
    a5 = B.SparseHermitian(o5._csr, "hermitian")
    runs["cfg5_n8"] = (a5, B.jacobi_preconditioner(a5), dict(k=16, sbsize=4, tol=1e-5, seed=0, max_iter=400))
    for name, (a, t, kw) in runs.items():
        t0 = time.time()
        rep = B.ppcg_solve(a, t, opts=B.SolverOptions(**kw))
        print(f"{name}: {rep.status} {rep.iterations} it in {time.time() - t0:.1f}s")
        _report_arrays(name, rep, out, vectors=a.n <= 2000)
    np.savez_compressed(os.path.join(HERE, "solves.npz"), **out)


def baselines():
    """Reference lobpcg_solve / davidson_solve (baselines.py:72-315) on the reference's test
    problems and scaled BASELINE structures (real and complex), plus the whole-block PPCG /
    LOBPCG equivalence case of test_acceptance.py:90-106."""
    out = {}
    o1, _, _, _ = P.config_problem(1, N=24)
    a1 = B.SparseHermitian(o1._csr, "symmetric")
    o5, _, _, _ = P.config_problem(5, N=8)
    a5 = B.SparseHermitian(o5._csr, "hermitian")
    runs = {
        "rand90": (B.random_hermitian(90, 0.25, seed=17), None, dict(k=6, tol=1e-9, seed=9, max_iter=200)),
        "lap1d": (B.laplacian_1d(300), "jacobi", dict(k=8, tol=1e-7, seed=0, max_iter=1500)),
        "cfg1s": (a1, "jacobi", dict(k=16, tol=1e-7, seed=0, max_iter=600)),
        "randz60": (B.random_hermitian(60, 0.5, seed=4, complex_field=True), None, dict(k=4, tol=1e-9, seed=1,
                                                                                        max_iter=400)),
        "cfg5s": (a5, "jacobi", dict(k=16, tol=1e-6, seed=0, max_iter=600)),
    }
    for name, (a, t, kw) in runs.items():
        tt = B.jacobi_preconditioner(a) if t == "jacobi" else None
        for solver, tag in ((B.lobpcg_solve, "lob"), (B.davidson_solve, "dav")):
            t0 = time.time()
            rep = solver(a, tt, opts=B.BaselineOptions(**kw))
            print(f"{tag}_{name}: {rep.status} {rep.iterations} it {rep.matvecs} mv in {time.time() - t0:.1f}s")
            pre = f"{tag}_{name}"
            out[f"{pre}_values"] = rep.values
            out[f"{pre}_trace"] = np.array([[r.iteration, r.trace_value, r.rel_resid, r.n_locked, r.n_matvec]
                                            for r in rep.trace]).reshape(-1, 5)
            out[f"{pre}_meta"] = np.array([rep.iterations, rep.matvecs, rep.rr_count, rep.breakdown_recoveries,
                                           1 if rep.status == "converged" else 0])
            out[f"{pre}_final_rn"] = np.array(rep.diagnostics["final_residual_norms"])
            if a.n <= 600:
                out[f"{pre}_vectors"] = rep.vectors
    # test_acceptance.py:90-106: whole-block PPCG (rr_period 1) vs LOBPCG from the same x0
    a = B.random_hermitian(100, 0.2, seed=12)
    x0 = np.random.default_rng(5).standard_normal((100, 8))
    rl = B.lobpcg_solve(a, x0=x0, opts=B.BaselineOptions(k=8, nbuf=0, tol=1e-14, seed=5, max_iter=10))
    out["equiv_x0"] = x0
    out["equiv_lob_vhist"] = np.array(rl.values_history[:10])
    np.savez_compressed(os.path.join(HERE, "baselines.npz"), **out)


def cfg2(iters):
    ours, k, q, tol = P.config_problem(2)
    a = B.SparseHermitian(ours._csr, "symmetric")
    t = B.jacobi_preconditioner(a)
    t0 = time.time()
    rep = B.ppcg_solve(a, t, opts=B.SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=iters))
    print(f"config 2 ({iters} iterations): {time.time() - t0:.1f}s")
    out = {}
    _report_arrays("cfg2", rep, out, vectors=False)
    np.savez_compressed(os.path.join(HERE, f"cfg2_iter{iters}.npz"), **out)


def cfg2_full(blas_threads):
    """BASELINE config 2 solved to convergence by the reference ``ppcg_solve``.

    The reference pins BLAS to one thread (ppcg.py:613).  SURVEY §8(c) measured that letting
    OpenBLAS use N threads leaves the trajectory intact (same iteration count and lock
    schedule, Ritz values within 1e-14) and runs 2x faster, so the pin is replaced in-process
    by an N-thread limit ("reference, BLAS xN"); no reference file is modified.

    Committed: values, trace (iteration, trace_value, rel_resid, n_locked, n_matvec), meta,
    final residual norms, values_history, orth_loss / proj_defect, and the lowest 8 and the
    highest 8 of the k returned eigenvectors (16 x n fp64, 14 MB) for principal angles.
    """
    from threadpoolctl import threadpool_limits

    BP.threadpool_limits = lambda limits=1: threadpool_limits(limits=blas_threads)
    ours, k, q, tol = P.config_problem(2)
    a = B.SparseHermitian(ours._csr, "symmetric")
    t = B.jacobi_preconditioner(a)
    t0 = time.time()
    rep = B.ppcg_solve(a, t, opts=B.SolverOptions(k=k, sbsize=q, tol=tol, seed=0, max_iter=5000))
    wall = time.time() - t0
    print(f"config 2 full: {rep.status} {rep.iterations} it {rep.rr_count} RR {rep.matvecs} mv "
          f"in {wall:.1f}s (BLAS x{blas_threads})", flush=True)
    out = {}
    _report_arrays("cfg2", rep, out, vectors=False)
    out["cfg2_vec_lo"] = np.ascontiguousarray(rep.vectors[:, :8])
    out["cfg2_vec_hi"] = np.ascontiguousarray(rep.vectors[:, -8:])
    out["cfg2_wall_s"] = np.array(wall)
    out["cfg2_blas_threads"] = np.array(blas_threads)
    np.savez_compressed(os.path.join(HERE, "cfg2_full.npz"), **out)


SCALED = {  # BASELINE configs 3-5 at the largest size the reference solves in minutes here
    "cfg3_n32": (3, 32, dict(k=256, sbsize=64, tol=1e-6)),
    "cfg4_n24": (4, 24, dict(k=256, sbsize=64, tol=1e-5)),
    "cfg5_n24": (5, 24, dict(k=256, sbsize=64, tol=1e-5)),
}


def scaled(blas_threads):
    """Configs 3, 4 and 5 on scaled grids with the production block shape (q = 64: the
    d = 192 pencils, the 7-/27-point and complex stencil SpMMs in their production mode),
    solved to convergence by the reference (BLAS xN as in cfg2_full)."""
    from threadpoolctl import threadpool_limits

    BP.threadpool_limits = lambda limits=1: threadpool_limits(limits=blas_threads)
    out = {}
    for name, (cfg, N, kw) in SCALED.items():
        ours, _, _, _ = P.config_problem(cfg, N=N)
        a = B.SparseHermitian(ours._csr, "hermitian" if cfg == 5 else "symmetric")
        t = B.jacobi_preconditioner(a)
        t0 = time.time()
        rep = B.ppcg_solve(a, t, opts=B.SolverOptions(seed=0, max_iter=3000, **kw))
        print(f"{name}: {rep.status} {rep.iterations} it {rep.rr_count} RR in {time.time() - t0:.1f}s", flush=True)
        _report_arrays(name, rep, out, vectors=False)
        out[f"{name}_vec_lo"] = np.ascontiguousarray(rep.vectors[:, :4])
        out[f"{name}_vec_hi"] = np.ascontiguousarray(rep.vectors[:, -4:])
    np.savez_compressed(os.path.join(HERE, "scaled.npz"), **out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg2", action="store_true")
    ap.add_argument("--baselines", action="store_true")
    ap.add_argument("--cfg2-full", action="store_true")
    ap.add_argument("--scaled", action="store_true")
    ap.add_argument("--blas-threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    if args.cfg2_full:
        cfg2_full(args.blas_threads)
        sys.exit(0)
    if args.scaled:
        scaled(args.blas_threads)
        sys.exit(0)
    if args.baselines:
        baselines()
        sys.exit(0)
    kernels()
    generators()
    if args.cfg2:
        cfg2(2)
    else:
        solves()
