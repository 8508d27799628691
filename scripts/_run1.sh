#!/bin/bash
export TSD_LIB=$PWD/ab/libUS.so
for g in c2.json c3s.json c4.json c5s.json; do echo $g; timeout 900 python scripts/cmp_golden.py $g 2>&1 | tail -1; done
timeout 900 python -m pytest -q -x tests/test_api_phases.py 2>&1 | tail -1
unset TSD_LIB
timeout 900 python scripts/ab.py c4 ab/libH.so ab/libUS.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c5 ab/libH.so ab/libUS.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c2 ab/libH.so ab/libUS.so 2>&1 | tail -2
for L in H US; do export TSD_LIB=$PWD/ab/lib$L.so; timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_next_length" -s 100 -c 1 python scripts/one_run.py c4 130 2>&1 | grep -E "gpu__time|dram__"; done
