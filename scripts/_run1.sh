cd $GRAFT_REPO_ROOT
python scripts/tune.py c3 rc_min_m=100000,256,384,512 2>&1 | tail -4
python scripts/tune.py c5 rc_min_m=100000,256,384,512 2>&1 | tail -4
python scripts/tune.py c4 rc_min_m=100000,384 2>&1 | tail -2
