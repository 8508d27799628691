#!/bin/bash
export TSD_LIB=$PWD/ab/libPKB.so
timeout 900 python scripts/cmp_golden.py c4.json 2>&1 | tail -1
unset TSD_LIB
timeout 900 python scripts/ab.py c4 ab/libLP.so ab/libPKB.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c5 ab/libLP.so ab/libPKB.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c2 ab/libLP.so ab/libPKB.so 2>&1 | tail -2
