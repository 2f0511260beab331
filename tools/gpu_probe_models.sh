# the 8B-shape live runs alone, with their run outputs in the reference schema
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_model8b.py -q -x --timeout=400 -p no:cacheprovider 2>&1 | tail -2
timeout 900 python tools/c2_model_probe.py > gpurun_out/c2_model.json 2>gpurun_out/c2_model.err; echo c2m=$?
timeout 900 python tools/c4_model_probe.py > gpurun_out/c4_model.json 2>gpurun_out/c4_model.err; echo c4m=$?
python -c "
import json
for f in ('c2_model', 'c4_model'):
    d=json.load(open(f'gpurun_out/{f}.json')); print(f, d['trace_metrics'], d['pause'], d['switch_step'], d['tokens_equal_static'])"
ls gpurun_out/c2_model_run gpurun_out/c4_model_run
