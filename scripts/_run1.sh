cd $GRAFT_REPO_ROOT
python scripts/cmp_golden.py c4.json
python scripts/cmp_golden.py c3.json
python scripts/cmp_golden.py c2.json
for c in c4 c5 c3 c2; do python scripts/tune.py $c wit_cache=1 2>&1 | tail -1; done
