cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider 2>&1 | tail -5
timeout 600 python tools/time_attn.py 2>&1 | tail -5
