cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -x 2>&1 | tail -2
AB="14=1|14=0" ROUNDS=3 timeout 900 python tools/ab_terms.py vlarge 1 2>&1 | tail -3
