#!/bin/bash
out=gpurun_out
timeout 600 python scripts/cmp_golden.py c4.json 2>&1 | tail -1
timeout 600 python scripts/cmp_golden.py c2.json 2>&1 | tail -1
timeout 900 python scripts/ab.py c4 ab/libBASE.so ab/libW2.so ab/libW3.so 2>&1 | tail -3
timeout 600 python scripts/ab.py c2 ab/libBASE.so ab/libW2.so ab/libW3.so 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum -k regex:"k_witness_list" -s 9 -c 4 python scripts/one_run.py c4 12 2>&1 | grep -E "k_witness_list|gpu__time" | head -8
