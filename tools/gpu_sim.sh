cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_simulation.py -q -p no:cacheprovider --timeout=600 2>&1 | tail -40
