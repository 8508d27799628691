cd $GRAFT_REPO_ROOT
python scripts/cmp_golden.py c4.json
python scripts/cmp_golden.py c3.json
python scripts/tune.py c4 band0_sides=1,2 2>&1 | tail -2
python scripts/tune.py c2 band0_sides=1,2 2>&1 | tail -2
python scripts/tune.py c3 band0_sides=1,2 2>&1 | tail -2
python scripts/tune.py c5 band0_sides=1,2 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/l_c4_w4.csv python scripts/one_run.py c4 24 > gpurun_out/l_c4_w4.txt 2>&1
