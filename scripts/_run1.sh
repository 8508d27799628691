#!/bin/bash
timeout 900 python scripts/tune.py c4 band_fill=0,12,16,32,48 2>&1 | tail -5
