"""Summarises an ncu HBM capture (scripts/ncu_hbm.sh) of the statistics and
bitmap passes: per kernel the median launch time, the cold-cache DRAM bytes
ncu measured, the ALGORITHMIC bytes of one launch (the per-element figures
below x the elements one launch processes), and achieved = algorithmic / time
against the measured HBM peak (MEASURED_PEAKS.json hbm_gbs).

    python scripts/hbm_summary.py gpurun_out/hbm_c4_r02.csv c4 > profiles/r02_hbm_c4.txt

DRAM writes read as ~0 for most kernels: the written arrays stay in the 126 MB
L2 when the kernel ends (write-back happens later), so the DRAM column
undercounts writes; the algorithmic column counts them.
"""
import csv
import json
import os
import statistics
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402

KW = 1152


def per_launch_bytes(kernel, n, m):
    """Algorithmic bytes of one launch (element counts at the config's first lengths)."""
    N = n - m + 1
    if kernel == "k_next_length":
        # mu, sigma in (16) + t (8) + double-double prefix sums P1, P2 (32) in;
        # mu, sigma out (16) + df, dg, nrm (12) out; resident seed rows read + written
        L = 512 if N >= 148 * 6 * 512 * 4 // 5 else 256
        nb = 2 * ((N + L - 1) // L)
        return 84 * (N - 1) + 16 * nb * KW, f"84 B x {N - 1} windows + 16 B x {nb}x{KW} seed entries"
    if kernel == "k_derive":
        return 68 * N, f"68 B x {N} windows (mu, sigma, t, P1, P2 in; df, dg, nrm out)"
    if kernel == "k_try_init":
        return 21 * N, f"21 B x {N} rows (alive 1, ymax 4, emax 4, ythr 4, nnkey 8 written)"
    if kernel == "k_compact_group":
        return 5 * N, f"<= 5 B x {N} rows (1 B flag read, 4 B list entry per live row)"
    if kernel == "k_init_finish":
        return 32 * N, f"32 B x {N} windows (sums in, mu, sigma out)"
    if kernel == "k_init_prefix":
        return 24 * N, f"24 B x {N} (t in, running sums out; one sequential thread per sum)"
    if kernel == "k_dd_chunk_sums":
        return 8 * n, f"8 B x {n} samples"
    if kernel == "k_dd_chunk_scan":
        return 40 * n, f"40 B x {n} samples (t in, two double-double prefixes out)"
    if kernel == "k_dd_scan_totals":
        return 0, "one thread, chunk totals"
    return 0, "?"


def main(path, cfg):
    n, _, m, _, _, _ = CONFIGS[cfg]
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    hdr, agg = None, defaultdict(lambda: defaultdict(list))
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = d["Kernel Name"].split("(")[0].split("<")[0]
            agg[k][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
    print(f"# {cfg}: n={n}, first length m={m}; ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
          f"dram__bytes_write.sum (cold cache, serialised); peak {peak} GB/s (MEASURED_PEAKS.json hbm_gbs)")
    print(f"{'kernel':18s} {'launches':>8s} {'median us':>10s} {'DRAM rd MB':>10s} {'DRAM wr MB':>10s} "
          f"{'alg MB':>8s} {'alg GB/s':>9s} {'frac':>6s}  algorithmic bytes")
    for k, v in agg.items():
        t = statistics.median(v["gpu__time_duration.sum"])  # ns
        rd = statistics.median(v["dram__bytes_read.sum"]) / 1e6
        wr = statistics.median(v["dram__bytes_write.sum"]) / 1e6
        b, how = per_launch_bytes(k, n, m)
        gbs = b / t if t > 0 else 0.0  # bytes / ns = GB/s
        print(f"{k:18s} {len(v['gpu__time_duration.sum']):8d} {t / 1e3:10.1f} {rd:10.2f} {wr:10.2f} "
              f"{b / 1e6:8.1f} {gbs:9.0f} {gbs / peak:6.2f}  {how}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
