#!/bin/bash
for g in c1.json c2.json c3s.json c4.json c5s.json small.json; do timeout 900 python scripts/cmp_golden.py $g 2>&1 | tail -1; done
timeout 2000 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
