#!/bin/bash
timeout 900 python scripts/tune.py c4 half_pk=20,22,23 2>&1 | tail -3
timeout 900 python scripts/tune.py c5 half_pk=20,22,23 2>&1 | tail -3
timeout 900 python scripts/tune.py c2 half_pk=20,22,23 2>&1 | tail -3
