#!/bin/bash
export TSD_LIB=$PWD/ab/libLP.so
for g in c1.json c2.json c3s.json c4.json c5s.json; do echo $g; timeout 900 python scripts/cmp_golden.py $g 2>&1 | tail -1; done
unset TSD_LIB
timeout 900 python scripts/ab.py c4 ab/libG.so ab/libLP.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c5 ab/libG.so ab/libLP.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c3 ab/libG.so ab/libLP.so 2>&1 | tail -2
timeout 900 python scripts/ab.py c2 ab/libG.so ab/libLP.so 2>&1 | tail -2
