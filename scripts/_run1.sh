cd $GRAFT_REPO_ROOT
python scripts/cmp_golden.py c4.json
python scripts/cmp_golden.py c3.json
for c in c4 c3 c5 c2; do python scripts/tune.py $c pass0_pk=0,1 2>&1 | tail -2; done
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
