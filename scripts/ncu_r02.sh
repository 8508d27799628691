#!/bin/bash
# r02 captures: launch lists (C2 full run, C4 first 16 lengths) and full ncu
# sections of the length step (k_next_length, C4) and of C2's scans.
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $out/launches_c2_$tag.csv python scripts/one_run.py c2 > /dev/null 2>&1; echo "ncu list c2 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $out/launches_c4_$tag.csv python scripts/one_run.py c4 16 > /dev/null 2>&1; echo "ncu list c4 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_next_length" -s 2 -c 2 \
   -o $out/next_length_c4_$tag -f python scripts/one_run.py c4 6 > /dev/null 2>&1; echo "ncu full next_length rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_compact|k_survivors" -s 40 -c 12 \
   -o $out/scan_c2_$tag -f python scripts/one_run.py c2 12 > /dev/null 2>&1; echo "ncu full c2 rc=$?"
