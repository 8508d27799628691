cd $GRAFT_REPO_ROOT
python scripts/cmp_golden.py c2.json
for c in c2 c4; do python scripts/tune.py $c track_chunks=1,2,3 2>&1 | tail -3; done
