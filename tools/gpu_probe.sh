cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_model8b.py -q -x --timeout=400 -p no:cacheprovider 2>&1 | tail -3
timeout 900 python tools/c4_model_probe.py > gpurun_out/c4_model.json 2>gpurun_out/c4_model.err; echo c4m=$?
python -c "
import json; d=json.load(open('gpurun_out/c4_model.json')); print({k:d[k] for k in d if k not in ('lag_polls','config_end')})"
tail -3 gpurun_out/c4_model.err
