"""Per-launch table of key ncu metrics from a .ncu-rep (run here, no GPU)."""
import csv, subprocess, sys, io
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
keys = [("gpu__time_duration.sum", "us", 1e-3), ("dram__bytes_read.sum", "MB", None), ("dram__bytes_write.sum", "MB", None),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1), ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%", 1),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%", 1), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%", 1), ("launch__registers_per_thread", "regs", 1),
        ("launch__grid_size", "grid", 1)]
def conv(v, unit):
    x = float(v.replace(",", ""))
    if unit in ("Gbyte", "GB"): return x * 1e3
    if unit in ("Kbyte", "KB"): return x * 1e-3
    if unit in ("byte",): return x * 1e-6
    if unit == "Mbyte": return x
    if unit in ("msecond", "ms"): return x * 1e3
    if unit in ("usecond", "us"): return x
    if unit in ("nsecond", "ns"): return x * 1e-3
    return x
idx = {k: h.index(k) for k, _, _ in keys if k in h}
print(f"{'kernel':34s} " + " ".join(f"{lab:>8s}" for _, lab, _ in keys))
for r in rows[2:]:
    name = r[h.index("Kernel Name")].split("(")[0][:34]
    vals = []
    for k, lab, _ in keys:
        if k in idx:
            vals.append(f"{conv(r[idx[k]], u[idx[k]]):8.1f}")
        else:
            vals.append(f"{'-':>8s}")
    print(f"{name:34s} " + " ".join(vals))

# --json PATH: merge {kernel: dram bytes per launch (first launch of each kernel)}
# into PATH (profiles/ncu_traffic.json, read by bench.py for roofline.traffic)
if "--json" in sys.argv:
    import json, os
    path = sys.argv[sys.argv.index("--json") + 1]
    doc = json.load(open(path)) if os.path.exists(path) else {"source": "ncu --set full --clock-control none", "kernels": {}}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "").strip()
        if name in doc["kernels"] and doc["kernels"][name].get("rep") == os.path.basename(rep):
            continue
        rd = conv(r[idx["dram__bytes_read.sum"]], u[idx["dram__bytes_read.sum"]]) * 1e6
        wr = conv(r[idx["dram__bytes_write.sum"]], u[idx["dram__bytes_write.sum"]]) * 1e6
        doc["kernels"][name] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                                "us": conv(r[idx["gpu__time_duration.sum"]], u[idx["gpu__time_duration.sum"]]),
                                "rep": os.path.basename(rep)}
    json.dump(doc, open(path, "w"), indent=1)
