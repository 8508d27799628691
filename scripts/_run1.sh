#!/bin/bash
export TSD_LIB=$PWD/ab/libPK1.so
timeout 600 python scripts/cmp_golden.py c4.json 2>&1 | tail -1
timeout 600 python scripts/cmp_golden.py c2.json 2>&1 | tail -1
unset TSD_LIB
timeout 900 python scripts/ab.py c4 ab/libW2.so ab/libPK1.so 2>&1 | tail -3
timeout 900 python scripts/ab.py c4 ab/libW2.so ab/libPK1.so 2>&1 | tail -3
timeout 600 python scripts/ab.py c2 ab/libW2.so ab/libPK1.so 2>&1 | tail -3
timeout 900 python scripts/ab.py c5 ab/libW2.so ab/libPK1.so 2>&1 | tail -3
