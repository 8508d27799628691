cd $GRAFT_REPO_ROOT
python scripts/tune.py c4 pk_rows=320,352,384,416,448 2>&1 | tail -5
python scripts/tune.py c3 pk_rows=448,480,512 2>&1 | tail -3
python scripts/tune.py c5 pk_rows=448,480,512 2>&1 | tail -3
