#!/bin/bash
timeout 300 python scripts/tune.py c2 scan_events=1 2>&1 | tail -1
timeout 300 python scripts/tune.py c2 scan_events=1 collect_skip=0 2>&1 | tail -1
