cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
PROBE_DUMP_S=100 timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$i tools/ring_probe.py 64 2>&1 | grep -v "^\*\|OMP" | tail -2
done
PL_PATCH_SOCKET=1 PROBE_DUMP_S=100 timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 tools/ring_probe.py 64 2>&1 | grep -v "^\*\|OMP" | tail -2
nproc; cat /proc/loadavg
