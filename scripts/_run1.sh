#!/bin/bash
timeout 900 python scripts/tune.py c2 band_few_wit=0,2,8 2>&1 | tail -3
timeout 900 python scripts/tune.py c3 few_m=512,300,200 few_lo=8 2>&1 | tail -3
timeout 900 python scripts/tune.py c5 few_m=512,300 few_lo=8 2>&1 | tail -2
