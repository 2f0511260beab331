import sys, json
sys.path.insert(0, '.')
from paper_2604_12171_b200.perf import c5_sweep
for r in c5_sweep(0, block_sizes=(16, 128)):
    print(json.dumps(r))
