import sys, json; sys.path.insert(0, '.')
from paper_2604_12171_b200.perf import c3_live_resize
print(json.dumps(c3_live_resize(0)))
