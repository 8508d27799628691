#!/bin/bash
# Parity suite + C4 (default) and C2 bench lines.  Usage: bash scripts/gpu_verify.sh <tag>
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu_$tag.txt
timeout 1500 python -m pytest tests -q -m gpu -x > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"
tail -3 $out/pytest_gpu_$tag.log
timeout 600 python bench.py --steps 3 --warmup 3 > $out/bench_c4_$tag.log 2>&1; echo "bench c4 rc=$?"
tail -1 $out/bench_c4_$tag.log | cut -c1-600
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_c2_$tag.log 2>&1; echo "bench c2 rc=$?"
tail -1 $out/bench_c2_$tag.log | cut -c1-600
