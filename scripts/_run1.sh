cd $GRAFT_REPO_ROOT
python scripts/cmp_golden.py c2.json
python scripts/cmp_golden.py c4.json
python scripts/cmp_golden.py c3.json
for c in c2 c4 c3 c5; do python scripts/tune.py $c witness=1 2>&1 | tail -1; done
