"""Summaries of ncu outputs for profiles/: a launch list (--metrics ... --csv)
and one --set full capture (.ncu-rep), as small JSON files.

    python tools/summarize_ncu.py launches gpurun_out/launches.csv > profiles/x_launches.json
    python tools/summarize_ncu.py full gpurun_out/prof.ncu-rep > profiles/x_ncu_full.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    per = defaultdict(dict)
    for r in rows[1:]:
        per[(int(r[ix["ID"]]), r[ix["Kernel Name"]])][r[ix["Metric Name"]]] = (
            float(r[ix["Metric Value"]].replace(",", "")), r[ix["Metric Unit"]])
    agg = defaultdict(lambda: {"launches": 0, "time_us": 0.0, "dram_read_MB": 0.0, "dram_write_MB": 0.0})
    for (_, name), m in per.items():
        short = name.split("(")[0]
        a = agg[short]
        a["launches"] += 1
        t, u = m.get("gpu__time_duration.sum", (0.0, "us"))
        a["time_us"] += t * (1e-3 if u == "ns" else (1e3 if u == "ms" else 1.0))
        for key, out in (("dram__bytes_read.sum", "dram_read_MB"), ("dram__bytes_write.sum", "dram_write_MB")):
            v, u2 = m.get(key, (0.0, "MB"))
            scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "KB": 1e-3, "MB": 1.0}.get(u2, 1.0)
            a[out] += v * scale
    total = sum(a["time_us"] for a in agg.values())
    out = {}
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["time_us"]):
        n = a["launches"]
        out[k] = {"launches": n, "avg_us": round(a["time_us"] / n, 3),
                  "share_of_gpu_time": round(a["time_us"] / total, 4) if total else None,
                  "avg_dram_read_MB": round(a["dram_read_MB"] / n, 3),
                  "avg_dram_write_MB": round(a["dram_write_MB"] / n, 3)}
    return {"source": path, "note": "ncu --metrics gpu__time_duration.sum,dram__bytes_*.sum "
            "--clock-control none (serialised, cold-cache replays: compare shares, not absolutes)",
            "kernels": out}


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for k in WANT:
            if k in h:
                d[k] = f"{r[h.index(k)]} {u[h.index(k)]}".strip()
        stalls = {n.replace("smsp__pcsamp_warps_issue_stalled_", ""): r[i] for i, n in enumerate(h)
                  if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")}
        d["stall_samples"] = {k: int(float(v)) for k, v in stalls.items() if v and float(v) > 0}
        out.append(d)
    return {"source": path, "note": "ncu --set full --clock-control none --import-source on", "launches": out}


if __name__ == "__main__":
    kind, p = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(p) if kind == "launches" else full(p), indent=1))
