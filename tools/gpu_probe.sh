cd $GRAFT_REPO_ROOT
for v in d1 d2 d3 g1 g2 g3; do
case $v in g*) export PL_RECLAIM_RELEASE_GRACE_MS=0;; esac
timeout 600 python bench.py --steps 10 --warmup 3 --skip-c3 --skip-c2 --skip-sweep --skip-cpu > gpurun_out/e2e_$v.json 2>gpurun_out/e2e_$v.err; echo rc=$?
python -c "
import json; l=json.loads(open('gpurun_out/e2e_$v.json').read().strip().splitlines()[-1]); print('$v', l['value'], l['e2e']['value'], l['e2e']['ms_per_step'], l['e2e_real_kv_from_host']['value'])"
done
