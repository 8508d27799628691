#!/bin/bash
# HBM evidence for the statistics and bitmap passes (north_star: "achieved HBM
# GB/s against peak for the statistics and bitmap passes"): DRAM bytes and
# duration of every launch of the length step (k_next_length), the Eq. 4 init
# (k_init_prefix / k_init_finish), the double-double prefix sums (k_dd_*), the
# try reset (k_try_init) and the alive-flag compaction (k_compact_group), at C2
# and at C4 (first 8 lengths).  ncu flushes caches before every kernel, so the
# DRAM bytes are the cold-cache traffic of one launch.
# Usage (repo root, under gpurun): bash scripts/ncu_hbm.sh <tag>
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
K='regex:k_next_length|k_init_finish|k_init_prefix|k_try_init|k_compact_group|k_dd_|k_derive'
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k "$K" -c 400 --csv \
  --log-file $out/hbm_c2_$tag.csv python scripts/one_run.py c2 16 > /dev/null 2>&1; echo "ncu hbm c2 rc=$?"
timeout 900 ncu --metrics $M --clock-control none -k "$K" -c 400 --csv \
  --log-file $out/hbm_c4_$tag.csv python scripts/one_run.py c4 8 > /dev/null 2>&1; echo "ncu hbm c4 rc=$?"
