#!/bin/bash
timeout 900 python scripts/tune.py c5 few_m=256,384,512,700 2>&1 | tail -4
timeout 900 python scripts/tune.py c4 few_m=512 few_lo=1,2,4 2>&1 | tail -3
timeout 900 python scripts/tune.py c3 few_m=256,384,512 2>&1 | tail -3
