#!/usr/bin/env python
"""Summarise a round's ncu captures (tools/profile_round.sh output) into profiles/<round>/:
  - launches_<cfg>_summary.txt : per-kernel share of the bench command's launch list
  - ncu_<cfg>_kernels.json/.md : per hot kernel duration, DRAM bytes, throughputs, occupancy
  - profiles/latest_traffic.json : DRAM bytes per launch read by bench.py (roofline.traffic)
Usage: python tools/ncu_summary.py gpurun_out/prof profiles/r01 C2"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__inst_executed.sum": "instructions",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
}


def to_base(v, unit):
    v = float(v)
    return v * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9,
                "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1.0)


def kernel_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[-1]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for m, key in METRICS.items():
        if m in hdr:
            i = hdr.index(m)
            try:
                d[key] = to_base(vals[i].replace(",", ""), units[i]) if key in ("duration", "dram_read", "dram_write") \
                    else float(vals[i].replace(",", ""))
            except ValueError:
                d[key] = vals[i]
    d["dram_bytes"] = d.get("dram_read", 0.0) + d.get("dram_write", 0.0)
    return d


def launch_summary(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void unnamed>::", "").replace("void ", "")
        a = agg[name]
        a[0] += 1
        a[1] += to_base(d["Metric Value"], d["Metric Unit"])
    tot = sum(a[1] for a in agg.values())
    lines = [f"{'share':>6} {'total_us':>11} {'launches':>8} {'avg_us':>9}  kernel"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{t / tot * 100:5.1f}% {t * 1e6:11.1f} {n:8d} {t / n * 1e6:9.2f}  {k}")
    return "\n".join(lines) + "\n"


def main(src, dst, cfg):
    os.makedirs(dst, exist_ok=True)
    lp = os.path.join(src, "launches.csv")
    if os.path.exists(lp):
        with open(os.path.join(dst, f"launches_{cfg}_summary.txt"), "w") as f:
            f.write("# ncu --metrics gpu__time_duration.sum --clock-control none, bench.py --config "
                    f"{cfg} --steps 1 --warmup 3 (cold-cache, serialised: compare shares)\n")
            f.write(launch_summary(lp))
    kernels = {}
    for name in ("rhals_sweeps_kernel", "tc_xht_resid_w_kernel", "tc_xht_resid_kernel", "tc_resid_kernel", "metrics_kernel", "tc_xw_kernel", "tc_xtw_kernel", "xw_tma_kernel", "xtw_tma_kernel"):
        rep = os.path.join(src, f"{name}_{cfg}.ncu-rep")
        if os.path.exists(rep):
            kernels[name] = kernel_metrics(rep)
    with open(os.path.join(dst, f"ncu_{cfg}_kernels.json"), "w") as f:
        json.dump(kernels, f, indent=1)
    with open(os.path.join(dst, f"ncu_{cfg}_kernels.md"), "w") as f:
        f.write(f"# ncu --set full, one launch per kernel ({cfg})\n\n")
        f.write("| kernel | us | DRAM MB | DRAM GB/s | SM % | mem % | L1 % | occupancy % | regs | grid |\n|---|---|---|---|---|---|---|---|---|---|\n")
        for name, d in kernels.items():
            f.write(f"| {d['kernel'][:60]} | {d.get('duration', 0) * 1e6:.1f} | {d['dram_bytes'] / 1e6:.1f} | "
                    f"{d['dram_bytes'] / max(d.get('duration', 0), 1e-12) / 1e9:.0f} | {d.get('sm_pct', 0):.1f} | {d.get('mem_pct', 0):.1f} | "
                    f"{d.get('l1_pct', 0):.1f} | {d.get('occupancy_pct', 0):.1f} | {d.get('registers', 0):.0f} | "
                    f"{d.get('grid', 0):.0f} |\n")
    lt = os.path.join(os.path.dirname(os.path.abspath(dst)), "latest_traffic.json")
    try:
        allt = json.load(open(lt))
    except Exception:
        allt = {}
    sk = [kernels[k]["dram_bytes"] for k in ("tc_xw_kernel", "tc_xtw_kernel") if k in kernels] or \
         [kernels[k]["dram_bytes"] for k in ("xw_tma_kernel", "xtw_tma_kernel") if k in kernels]
    allt[cfg] = {"source": os.path.join(os.path.basename(dst), f"ncu_{cfg}_kernels.json"),
                 "sketch_bytes_per_launch": sum(sk) / len(sk) if sk else None,
                 "kernels": {k: v["dram_bytes"] for k, v in kernels.items()}}
    json.dump(allt, open(lt, "w"), indent=1)
    print(open(os.path.join(dst, f"ncu_{cfg}_kernels.md")).read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "C2")
