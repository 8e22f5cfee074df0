"""SpMM variants on the BASELINE operators: row gather vs column-slice tiled.

usage: python tools/spmm_sweep.py [cfg ...]   (default 2 3 4)
Prints one JSON line per (config, width, offset, variant): ms, algorithmic GB/s
(2 n m s + nnz (s + 4) + 4 (n + 1)), fraction of MEASURED_PEAKS hbm_gbs, and
whether the variant's result is bitwise equal to the row gather's.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_7506_b200 import _lib  # noqa: E402
from paper_1407_7506_b200.operators import as_device_operator  # noqa: E402
from paper_1407_7506_b200.problems import config_problem  # noqa: E402


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6554.6


VARIANTS = [int(v) for v in os.environ.get("SPMM_VARIANTS", "0,1,2").split(",")]


def main():
    cfgs = [int(c) for c in sys.argv[1:]] or [2, 3, 4]
    lib = _lib.load()
    peak = hbm_peak()
    for cfg in cfgs:
        kw = {"N": 64} if cfg == 5 else {}
        a, k, q, tol = config_problem(cfg, **kw)
        d = as_device_operator(a)
        cplx = str(a.dtype) == "complex128"
        dt = torch.complex128 if cplx else torch.float64
        s = 16 if cplx else 8
        kt = k + -(-k * 2 // 100)
        for m, off in ((kt, 0), (kt - 10, 10), (kt - 11, 11)):
            ld = (kt + 15) // 16 * 16  # the solver's 128-byte rows
            g = torch.Generator(device="cuda").manual_seed(1)
            xb = torch.randn(a.n, ld, dtype=dt, device="cuda", generator=g)
            yb = torch.zeros(a.n, ld, dtype=dt, device="cuda")
            x, y = xb[:, off:off + m], yb[:, off:off + m]
            byts = 2.0 * a.n * m * s + d.nnz * (s + 4) + 4 * (a.n + 1)
            ref = None
            names = {0: "row_gather", 1: "vec", 2: "march", 3: "vec_u1", 4: "vec_u1_mb2", 5: "vec_u2_mb2",
                     6: "vec_u4", 7: "vec_u1_mb3"}
            for variant in VARIANTS:
                lib.bk_spmm_set_variant({0: 0, 1: 2, 2: 2}.get(variant, variant))
                type(d).use_stencil = variant == 2
                d.apply_into(x, y)
                torch.cuda.synchronize()
                out = y.clone()
                if ref is None:
                    ref = out
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 20
                e0.record()
                for _ in range(reps):
                    d.apply_into(x, y)
                e1.record()
                e1.synchronize()
                ms = e0.elapsed_time(e1) / reps
                print(json.dumps({"cfg": cfg, "n": a.n, "nnz": d.nnz, "m": m, "col_offset": off,
                                  "variant": names[variant],
                                  "grid": getattr(d.stencil, "grid", None), "ms": round(ms, 4),
                                  "gbs": round(byts / ms / 1e6, 1), "frac_hbm": round(byts / ms / 1e6 / peak, 3),
                                  "bitwise_equal_to_gather": bool(torch.equal(out, ref))}), flush=True)
            del xb, yb, ref, out
        lib.bk_spmm_set_variant(2)
        type(d).use_stencil = True
        del d, a
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
