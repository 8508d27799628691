#!/bin/bash
out=gpurun_out; mkdir -p $out
for g in c2.json c3s.json c4.json; do timeout 600 python scripts/cmp_golden.py $g 2>&1 | tail -2; done
timeout 900 python scripts/ab.py c4 ab/libSP0.so ab/libSP1.so 2>&1 | tail -3
timeout 600 python scripts/ab.py c2 ab/libSP0.so ab/libSP1.so 2>&1 | tail -3
timeout 900 python scripts/ab.py c5 ab/libSP0.so ab/libSP1.so 2>&1 | tail -3
