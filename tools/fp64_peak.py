"""Measure the FP64 roofline denominators on the box: cuBLAS DGEMM (torch.matmul fp64)
burst and sustained, plus the DMMA/DFMA probes of tools/fp64_peak.cu.  Writes one JSON
object to stdout; the committed copy lives in profiles/fp64_peak_r01.json."""
import json, subprocess, sys, time, os
import torch

def dgemm(n=8192, reps=10, sustain_s=4.0):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    burst = 2 * n**3 / best / 1e9
    t0 = time.time(); cnt = 0
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < sustain_s:
        c = a @ b; cnt += 1
        if cnt % 8 == 0: torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    sust = 2 * n**3 * cnt / e0.elapsed_time(e1) / 1e9
    return burst, sust

def tall_gram(n=110592, m=523):
    x = torch.randn(n, m, dtype=torch.float64, device="cuda")
    g = x.T @ x; torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); g = x.T @ x; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    gram = 2 * n * m * m / best / 1e9
    gm = torch.randn(m, m, dtype=torch.float64, device="cuda")
    y = x @ gm; torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); y = x @ gm; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    upd = 2 * n * m * m / best / 1e9
    return gram, upd

if __name__ == "__main__":
    res = {"gpu": torch.cuda.get_device_name(0)}
    b, s = dgemm()
    res["cublas_dgemm_8192_burst_tflops"] = round(b, 2)
    res["cublas_dgemm_8192_sustained_tflops"] = round(s, 2)
    g, u = tall_gram()
    res["cublas_tall_gram_110592x523_tflops"] = round(g, 2)
    res["cublas_tall_update_110592x523x523_tflops"] = round(u, 2)
    exe = sys.argv[1] if len(sys.argv) > 1 else None
    if exe:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=300).stdout
        res["probes"] = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
    print(json.dumps(res))
