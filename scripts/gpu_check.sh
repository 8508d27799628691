#!/bin/bash
# One GPU round: parity tests, bench, launch list and a full ncu capture of k_scan.
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [config] [tag]
cfg=${1:-c2}; tag=${2:-r01}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu_$tag.txt
timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"
tail -3 $out/pytest_gpu_$tag.log
timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 > $out/bench_${cfg}_$tag.log 2>&1; echo "bench rc=$?"
tail -1 $out/bench_${cfg}_$tag.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
   --log-file $out/launches_${cfg}_$tag.csv python bench.py --config $cfg --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 20 -c 3 \
   -o $out/scan_${cfg}_$tag -f python bench.py --config $cfg --steps 1 --warmup 0 --no-cpu-baseline > $out/ncu_full_$tag.log 2>&1
echo "ncu full rc=$?"
