"""Summarise ncu --set full captures of the emulated-FP64 kernels into JSON (per-launch dram
bytes, duration, tensor-pipe / shared-memory-path activity).  usage: ncu_ozaki_summary.py rep..."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ms_x1e-3",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "tc_smem_wavefronts_pct",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "mem_tensor_active_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-3, "ms": 1.0, "ns": 1e-6, "usecond": 1e-3,
        "msecond": 1.0, "nsecond": 1e-6}
out = {}
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").strip()
        d = {}
        for k, short in KEYS.items():
            cands = [j for j, x in enumerate(h) if x == k or x.endswith("." + k)]
            if cands:
                i = cands[0]
                v = float(r[i].replace(",", "")) if r[i] else None
                if v is not None and units[i] in UNIT:
                    v *= UNIT[units[i]]
                d[short.replace("_x1e-3", "") if k.startswith("gpu__time") else short] = v
        if d.get("dram_read") is not None:
            d["dram_bytes_per_launch"] = d["dram_read"] + (d.get("dram_write") or 0)
        out.setdefault(name, []).append(d)
print(json.dumps({"source": "ncu --set full --clock-control none (tools/oz_one.py on config-2 shapes)",
                  "kernels": out}, indent=1))
