cd $GRAFT_REPO_ROOT
timeout 1200 python tools/sweep_lm.py vlarge 8 "5=83886080|5=67108864|5=58720256|5=50331648|5=100663296" 2>&1 | tail -10
