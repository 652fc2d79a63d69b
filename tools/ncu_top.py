"""Summarize an ncu report: key metrics + top stalled SASS lines (run here, no GPU)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print("kernel:", name[:80])
    for k in keys:
        if k in hdr:
            i = hdr.index(k)
            print(f"  {k:70s} {r[i]:>14s} {units[i]}")
if len(sys.argv) > 2:
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                           "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(sass)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]
    sc = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    col = idx["Warp Stall Sampling (All Samples)"]
    tot = sum(int(r[col] or 0) for r in data)
    print("samples", tot)
    agg = {}
    for r in data:
        for c in sc:
            agg[c] = agg.get(c, 0) + int(r[idx[c]] or 0)
    print(sorted(agg.items(), key=lambda x: -x[1])[:10])
    for r in sorted(data, key=lambda r: -int(r[col] or 0))[:int(sys.argv[2])]:
        st = sorted(((int(r[idx[c]] or 0), c) for c in sc), reverse=True)[:2]
        print(f"{int(r[col] or 0):7d} {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:58]:58s} {st}")
