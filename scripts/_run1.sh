#!/bin/bash
export TSD_LIB=$PWD/ab/libNL2.so
timeout 600 python scripts/cmp_golden.py c4.json 2>&1 | tail -1
timeout 900 python -m pytest -q -x tests/test_api_phases.py 2>&1 | tail -1
for L in NL1 NL2; do
export TSD_LIB=$PWD/ab/lib$L.so
timeout 900 ncu --metrics gpu__time_duration.sum -k regex:"k_next_length" -s 100 -c 3 python scripts/one_run.py c4 130 2>&1 | grep -E "gpu__time"
done
unset TSD_LIB
timeout 900 python scripts/ab.py c4 ab/libNL1.so ab/libNL2.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c2 ab/libNL1.so ab/libNL2.so 2>&1 | tail -2
