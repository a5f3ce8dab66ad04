cd $GRAFT_REPO_ROOT
PV_PARITY_REPORT=gpurun_out/parity_loop.json timeout 600 python -m pytest tests/test_gpu_loopback.py -m gpu -q -s 2>&1 | tail -10
