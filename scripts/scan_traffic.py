"""DRAM traffic per scan launch (bench.py's roofline.traffic) from an ncu CSV:
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_scan|k_band0" --csv \
    --log-file X.csv python scripts/one_run.py <cfg> [lengths]
python scripts/scan_traffic.py X.csv <cfg> "<how>" > profiles/scan_traffic_<cfg>.json"""
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iN, iV, iK, iI = h.index("Metric Name"), h.index("Metric Value"), h.index("Kernel Name"), h.index("ID")
rd, wr, ids = 0.0, 0.0, set()
unit = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
iU = h.index("Metric Unit")
for r in rows[1:]:
    if "k_scan" not in r[iK] and "k_band0" not in r[iK]:
        continue
    ids.add(r[iI])
    v = float(r[iV].replace(",", "")) * unit.get(r[iU], 1.0)
    if r[iN] == "dram__bytes_read.sum":
        rd += v
    elif r[iN] == "dram__bytes_write.sum":
        wr += v
n = len(ids)
print(json.dumps({"kernel": "k_scan / k_band0_pair", "launches": n, "bytes_per_launch": (rd + wr) / max(n, 1),
                  "dram_read_bytes": rd, "dram_write_bytes": wr, "how": sys.argv[3]}, indent=1))
