"""SpMM kernel comparison on the BASELINE operators: vector gather, offset-ELL march
(bk_spmm_march_*) and the stencil-slot kernel variants (bk_spmm_stencil_*).

usage: python tools/stencil_sweep.py [cfg ...]   (default 2 3 4 5; config 5 at 64^3, one GPU)
One JSON line per (config, column offset, kernel): ms, algorithmic GB/s (2 n m s + nnz (s + 4)
+ 4 (n + 1)), fraction of MEASURED_PEAKS hbm_gbs, bitwise equality to the gather.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1407_7506_b200 import _lib  # noqa: E402
from paper_1407_7506_b200.operators import DeviceCsr  # noqa: E402
from paper_1407_7506_b200.problems import config_problem  # noqa: E402


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6554.6


# stencil-slot configurations (bk_spmm_stencil_set_config): v (variant), 10 + v (slice-fastest
# unit order), 20 + v (tile-fastest unit order)
SLOT_CFGS = [int(c) for c in os.environ.get("SLOT_CFGS", "0,1,10,20,21").split(",")]


def main():
    cfgs = [int(c) for c in sys.argv[1:]] or [2, 3, 4, 5]
    lib = _lib.load()
    peak = hbm_peak()
    for cfg in cfgs:
        kw = {"N": 64} if cfg == 5 else {}
        a, k, q, tol = config_problem(cfg, **kw)
        DeviceCsr.stencil_kinds = ("slot", "march")
        d = DeviceCsr(a._csr)
        plan = d.stencil
        cplx = d.complex
        dt = torch.complex128 if cplx else torch.float64
        s = 16 if cplx else 8
        kt = k + -(-k * 2 // 100)
        ld = (kt + 15) // 16 * 16
        g = torch.Generator(device="cuda").manual_seed(1)
        xb = torch.randn(a.n, ld, dtype=dt, device="cuda", generator=g)
        yb = torch.zeros(a.n, ld, dtype=dt, device="cuda")
        for m, off in ((kt, 0), (kt - 11, 11)):
            x, y = xb[:, off:off + m], yb[:, off:off + m]
            byts = 2.0 * a.n * m * s + d.nnz * (s + 4) + 4 * (a.n + 1)
            ref = None
            variants = [("vec", False, False, 0), ("march", True, False, 0)]
            variants += [(f"slot{c}", True, True, c) for c in SLOT_CFGS]
            for name, stencil, slot, cfgv in variants:
                DeviceCsr.use_stencil = stencil
                plan.use_slot = slot
                lib.bk_spmm_stencil_set_config(cfgv)
                y.zero_()
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
                print(json.dumps({"cfg": cfg, "n": a.n, "nnz": d.nnz, "st": plan.st, "m": m, "col_offset": off,
                                  "kernel": name, "ms": round(ms, 4), "gbs": round(byts / ms / 1e6, 1),
                                  "frac_hbm": round(byts / ms / 1e6 / peak, 3),
                                  "bitwise_equal_to_gather": bool(torch.equal(out, ref))}), flush=True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            y.copy_(x)
            e0.record()
            for _ in range(20):
                y.copy_(x)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1) / 20
            print(json.dumps({"cfg": cfg, "m": m, "col_offset": off, "kernel": "copy (same block, torch)",
                              "ms": round(ms, 4), "gbs_spmm_bytes": round(byts / ms / 1e6, 1),
                              "frac_hbm": round(byts / ms / 1e6 / peak, 3)}), flush=True)
            del ref, out
        lib.bk_spmm_stencil_set_config(0)
        DeviceCsr.use_stencil = True
        plan.use_slot = True
        del d, a, xb, yb, plan
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
