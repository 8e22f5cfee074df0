"""Summarise ncu captures (.ncu-rep, --set full) and launch lists into profiles/.

  python tools/ncu_summary.py OUT.json rep1.ncu-rep [rep2.ncu-rep ...] [--launches launches.csv]

Per kernel: duration, DRAM read+write bytes (the roofline `traffic`), tensor/FP64 pipe
activity, occupancy, top stall reasons.  The launch list gives each kernel's share of the
profiled run (cold-cache, serialised: compare shares, not absolutes).
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_ld_bank_conflicts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum": "smem_ld_wavefronts",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
        "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
TIME_UNITS = {"nsecond", "usecond", "msecond", "second", "ns", "us", "ms", "s"}


def rep_summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": re.sub(r"\(.*", "", vals[hdr.index("Kernel Name")])}
        stalls = {}
        for h, u, v in zip(hdr, units, vals):
            try:
                fv = float(v.replace(",", ""))
            except ValueError:
                continue
            if h in KEYS:
                name = KEYS[h]
                if u in UNIT:
                    fv *= UNIT[u]
                    name += "_ms" if u in TIME_UNITS else "_bytes"
                d[name] = fv
            m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", h)
            if m and fv > 0.05:
                stalls[m.group(1)] = round(fv, 3)
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        d["dram_bytes_per_launch"] = d.get("dram_read_bytes", 0) + d.get("dram_write_bytes", 0)
        res.append(d)
    return res


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r"\(.*", "", r[ki])[:80]
        tot[name] += float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        cnt[name] += 1
    T = sum(tot.values())
    return [{"kernel": k, "ms": round(v, 4), "share": round(v / T, 4), "launches": cnt[k]}
            for k, v in sorted(tot.items(), key=lambda kv: -kv[1])]


if __name__ == "__main__":
    out = sys.argv[1]
    args = sys.argv[2:]
    launches = None
    if "--launches" in args:
        i = args.index("--launches")
        launches = args[i + 1]
        args = args[:i] + args[i + 2:]
    # --roofline NAME=REP: all launches of REP form one roofline call (e.g. the Gram's main +
    # strip launch); kernels[NAME.split('_')[0] + '_kernel'] then carries their summed traffic
    roofs = []
    while "--roofline" in args:
        i = args.index("--roofline")
        roofs.append(args[i + 1].split("=", 1))
        args = args[:i] + args[i + 2:]
    summary = {"kernels": {}, "captures": []}
    for p in args:
        for d in rep_summary(p):
            summary["captures"].append(d)
            summary["kernels"].setdefault(d["kernel"].split("::")[-1].split("<")[0].replace("void ", ""), d)
    for name, rep in roofs:
        ls = rep_summary(rep)
        entry = {"launches": [{k: d.get(k) for k in ("kernel", "duration_ms", "dram_bytes_per_launch",
                                                      "tensor_pipe_active_pct", "grid")} for d in ls],
                 "dram_bytes_total": sum(d["dram_bytes_per_launch"] for d in ls),
                 "duration_ms_total": sum(d.get("duration_ms", 0.0) for d in ls), "rep": rep}
        summary["roofline_" + name] = entry
        key = name.split("_")[0] + "_kernel"
        base = dict(ls[0])
        base["dram_bytes_per_launch"] = entry["dram_bytes_total"]
        base["note"] = f"dram_bytes_per_launch = all launches of the roofline call roofline_{name}"
        summary["kernels"][key] = base
    if launches:
        summary["launch_shares"] = launch_shares(launches)
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps({k: {kk: v[kk] for kk in ("duration_ms", "dram_bytes_per_launch") if kk in v}
                      for k, v in summary["kernels"].items()}, indent=1))
