#!/bin/bash
export TSD_LIB=$PWD/ab/libNL1.so
timeout 600 python scripts/cmp_golden.py c4.json 2>&1 | tail -1
timeout 600 python scripts/cmp_golden.py c2.json 2>&1 | tail -1
timeout 900 python -m pytest -q -x tests/test_api_phases.py 2>&1 | tail -2
unset TSD_LIB
timeout 900 python scripts/ab.py c4 ab/libF.so ab/libNL1.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c2 ab/libF.so ab/libNL1.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c5 ab/libF.so ab/libNL1.so 2>&1 | tail -2
for L in F NL1; do
export TSD_LIB=$PWD/ab/lib$L.so
timeout 900 ncu --metrics gpu__time_duration.sum -k regex:"k_next_length" -s 20 -c 3 python scripts/one_run.py c4 30 2>&1 | grep -E "gpu__time"
done
