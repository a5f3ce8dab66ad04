cd $GRAFT_REPO_ROOT
AB="2=2|2=0|2=1|3=0|4=0" ROUNDS=2 timeout 900 python tools/ab_terms.py vlarge 1 2>&1 | tail -6
