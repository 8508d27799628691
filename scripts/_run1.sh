#!/bin/bash
export TSD_LIB=$PWD/ab/libPKONE.so
timeout 600 python scripts/cmp_golden.py c4.json 2>&1 | tail -1
unset TSD_LIB
timeout 900 python scripts/ab.py c4 ab/libPKONE.so ab/libPK1.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c4 ab/libPK1.so ab/libPKONE.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c3 ab/libPK1.so ab/libPKONE.so 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum -k regex:"k_band0_pk" -s 5 -c 3 python scripts/one_run.py c4 12 2>&1 | grep -E "gpu__time" 
export TSD_LIB=$PWD/ab/libPK1.so
timeout 900 ncu --metrics gpu__time_duration.sum -k regex:"k_band0_pk" -s 5 -c 3 python scripts/one_run.py c4 12 2>&1 | grep -E "gpu__time" 
