#!/bin/bash
# Full ncu sections (with source correlation) of one C4 try's scans: the paired
# band-0 walk, the later band passes, the full rows and the collection.  Skips
# the first try (all rows die in pass 0 at r = 2 sqrt(m)).
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_band0" -s 4 -c 6 \
   -o $out/scan_c4_$tag -f python scripts/one_run.py c4 3 > $out/ncu_full_c4_$tag.log 2>&1; echo "ncu full c4 rc=$?"
