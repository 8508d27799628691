#!/bin/bash
# Round-2 evidence: bench lines (C2..C5), the reference arm, launch lists of
# whole C2 / C4 discoveries and full ncu captures of the dominant kernels.
# Usage (repo root, under gpurun): bash scripts/gpu_evidence_r02.sh <tag>
tag=${1:-r02y}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu_$tag.txt
timeout 900 python bench.py --steps 5 --warmup 3 > $out/bench_c4_$tag.log 2>&1; echo "bench c4 rc=$?"
timeout 900 python bench.py --config c2 --steps 5 --warmup 3 > $out/bench_c2_$tag.log 2>&1; echo "bench c2 rc=$?"
for c in c3 c5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $out/bench_${c}_$tag.log 2>&1; echo "bench $c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $out/ref_c4_$tag.log 2>&1; echo "ref c4 rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $out/launches_c4_$tag.csv python scripts/one_run.py c4 > /dev/null 2>&1; echo "ncu list c4 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $out/launches_c2_$tag.csv python scripts/one_run.py c2 > /dev/null 2>&1; echo "ncu list c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"k_band0_pk|k_scan|k_witness$|k_next_length" -s 60 -c 12 \
   -o $out/full_c4_$tag -f python scripts/one_run.py c4 12 > /dev/null 2>&1; echo "ncu full c4 rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_$tag.log 2>&1; echo "smoke rc=$?"
