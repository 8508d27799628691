#!/bin/bash
# One GPU round: parity tests, bench lines (C2 default + C4), launch lists and a
# full ncu capture of the dominant k_scan launches.
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [tag]
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu_$tag.txt
timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"
tail -2 $out/pytest_gpu_$tag.log
timeout 600 python bench.py --steps 5 --warmup 3 > $out/bench_c2_$tag.log 2>&1; echo "bench c2 rc=$?"
tail -1 $out/bench_c2_$tag.log | cut -c1-400
timeout 900 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline > $out/bench_c4_$tag.log 2>&1
echo "bench c4 rc=$?"; tail -1 $out/bench_c4_$tag.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $out/launches_c2_$tag.csv python scripts/one_run.py c2 > /dev/null 2>&1
echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 0 -c 6 \
   -o $out/scan_c4_$tag -f python scripts/one_run.py c4 2 > $out/ncu_full_c4_$tag.log 2>&1
echo "ncu full c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 20 -c 8 \
   -o $out/scan_c2_$tag -f python scripts/one_run.py c2 12 > $out/ncu_full_c2_$tag.log 2>&1
echo "ncu full c2 rc=$?"
