"""Per-CUDA-source-line stall samples and executed instructions of an ncu report's
cuda,sass source view (run here, no GPU):  python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = defaultdict(lambda: [0, 0, defaultdict(int), ""])
files = {}
cur_file = "?"
hdr = None
line = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) - 2:
        continue
    if r[0]:
        line = (cur_file, int(r[0]), r[1].strip()[:70])
    if not r[2] or line is None:  # cuda line row without sass
        continue
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_e = hdr.index("Instructions Executed")
    try:
        s = int(r[i_s] or 0)
        e = int(r[i_e] or 0)
    except ValueError:
        continue
    a = agg[line]
    a[0] += s
    a[1] += e
    for j, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and j < len(r):
            try:
                a[2][h] += int(r[j] or 0)
            except ValueError:
                pass
tot = sum(a[0] for a in agg.values()) or 1
toti = sum(a[1] for a in agg.values()) or 1
print(f"samples {tot}, instructions {toti}")
for key, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    st = sorted(a[2].items(), key=lambda kv: -kv[1])[:2]
    print(f"{a[0] / tot * 100:5.1f}% {a[1] / toti * 100:5.1f}%i {key[0]}:{key[1]:<5d} {key[2]:70s} "
          + " ".join(f"{k[6:]}={v}" for k, v in st))
