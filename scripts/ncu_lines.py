"""Top source lines by warp-stall samples of one kernel in an ncu report:
python scripts/ncu_lines.py report.ncu-rep <launch-skip> [top]"""
import csv
import subprocess
import sys

rep, skip = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
fp, agg = None, {}
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        fp = r[1].split("/")[-1]
        continue
    if len(r) > 6 and r[0].isdigit() and r[2] == "-":
        k = (fp, int(r[0]))
        v = agg.get(k, (0, r[1][:90]))
        agg[k] = (v[0] + int(r[4]), v[1])
tot = sum(v[0] for v in agg.values()) or 1
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]:6d} {100 * v[0] / tot:5.1f}% {k[0]}:{k[1]} {v[1]}")
