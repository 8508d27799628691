#!/bin/bash
export TSD_LIB=$PWD/ab/libRC16.so
timeout 600 python scripts/cmp_golden.py c4.json 2>&1 | tail -1
timeout 600 python scripts/cmp_golden.py c5s.json 2>&1 | tail -1
unset TSD_LIB
timeout 900 python scripts/ab.py c4 ab/libBASE2.so ab/libRC16.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c5 ab/libBASE2.so ab/libRC16.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c3 ab/libBASE2.so ab/libRC16.so 2>&1 | tail -2
