import sys
sys.path.insert(0, '.')
import torch
from paper_2604_12171_b200.kvstore import KvStore
f = lambda: round(torch.cuda.mem_get_info(0)[0] / 1e9, 1)
print("start", f())
st = KvStore(2, 4, 16, 40000, (0, 1), num_groups=20, cell_bytes=4096)
print("after create 2 groups x 40000 units", f(), st.info()["mapped_bytes"] / 1e9)
st.close()
print("after close", f())
st = KvStore(2, 4, 16, 40000, (0, 1), num_groups=20, cell_bytes=4096)
st.drop_layer_groups([0])
print("after drop (deferred)", f(), st.vmm_stats())
st.reclaim()
print("after reclaim", f(), st.vmm_stats())
st.resize(20000)
print("after shrink (deferred)", f(), st.vmm_stats())
st.reclaim()
print("after reclaim", f(), st.vmm_stats())
del st
print("after del", f())
