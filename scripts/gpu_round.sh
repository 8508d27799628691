#!/bin/bash
# End-of-stretch evidence: parity suite, bench lines for C2 (default, with the
# reference CPU baseline), C3, C4, C5, launch lists and ncu captures.
# Usage (repo root, under gpurun): bash scripts/gpu_round.sh <tag>
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu_$tag.txt
timeout 900 python -m pytest tests -q -m gpu > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"
tail -1 $out/pytest_gpu_$tag.log
timeout 600 python bench.py --steps 5 --warmup 3 > $out/bench_c2_$tag.log 2>&1; echo "bench c2 rc=$?"
for c in c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > $out/bench_${c}_$tag.log 2>&1
  echo "bench $c rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $out/launches_c2_$tag.csv python scripts/one_run.py c2 > /dev/null 2>&1; echo "ncu list c2 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $out/launches_c4_$tag.csv python scripts/one_run.py c4 16 > /dev/null 2>&1; echo "ncu list c4 rc=$?"
# full capture: pass 0 and the next band passes of a working C4 try (skip the
# first, all-killing try: 3 launches), and 8 consecutive scans of C2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_band0" -s 8 -c 6 \
   -o $out/scan_c4_$tag -f python scripts/one_run.py c4 3 > $out/ncu_full_c4_$tag.log 2>&1; echo "ncu full c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_band0" -s 20 -c 8 \
   -o $out/scan_c2_$tag -f python scripts/one_run.py c2 12 > $out/ncu_full_c2_$tag.log 2>&1; echo "ncu full c2 rc=$?"
