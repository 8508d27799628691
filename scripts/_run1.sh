#!/bin/bash
for g in c2.json c4.json; do timeout 600 python scripts/cmp_golden.py $g 2>&1 | tail -1; done
timeout 900 python scripts/ab.py c4 ab/libBASE.so ab/libW1.so 2>&1 | tail -2
timeout 600 python scripts/ab.py c2 ab/libBASE.so ab/libW1.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c5 ab/libBASE.so ab/libW1.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c3 ab/libBASE.so ab/libW1.so 2>&1 | tail -2
