cd $GRAFT_REPO_ROOT
for v in 1 2; do
  PL_TRACE_RESIZE=1 timeout 400 python tools/c4_live.py > gpurun_out/c4_$v.json 2>gpurun_out/c4_$v.err; echo c4_$v=$?
  python -c "
import json; d=json.load(open('gpurun_out/c4_live.json')); print('$v', d['steps']['pause_ms'], json.dumps({r: v['post_commit'] for r, v in d['switch_phases_ms_by_rank'].items()}))"
  grep "drop_groups\|reclaim" gpurun_out/c4_$v.err | head -12
done
