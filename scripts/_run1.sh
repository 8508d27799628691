#!/bin/bash
timeout 600 python scripts/cmp_golden.py c4.json 2>&1 | tail -1
timeout 600 python scripts/cmp_golden.py c3s.json 2>&1 | tail -1
timeout 600 python scripts/cmp_golden.py c5s.json 2>&1 | tail -1
timeout 900 python scripts/tune.py c4 wit_wide=0,1 2>&1 | tail -2
timeout 900 python scripts/tune.py c4 wit_wide=0,1 2>&1 | tail -2
timeout 900 python scripts/tune.py c5 wit_wide=0,1 2>&1 | tail -2
timeout 900 python scripts/tune.py c3 wit_wide=0,1 2>&1 | tail -2
