"""Top SASS lines by warp-stall samples of an ncu report (profiling helper):
    python tools/ncu_sass_top.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
i_s, i_src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
i_ex = h.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for r in data) or 1
print("total warp instructions", sum(int(r[i_ex] or 0) for r in data))
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:n]:
    print(f"{float(r[i_s]) / tot * 100:5.1f}% ex={r[i_ex]:>9} {r[0][-5:]} {r[i_src][:100]}")
