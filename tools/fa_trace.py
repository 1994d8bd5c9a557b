"""clock64 trace of k_fa2's CTA 0 (softmax warp of each tile + MMA waits)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_19516_b200.device import lib
DEV = torch.device("cuda", 0)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
d, Hq, Hkv = 128, 32, 8
qkv = torch.randn(T, (Hq + 2 * Hkv) * d, device=DEV).to(torch.bfloat16)
q, k, v = qkv[:, :Hq * d], qkv[:, Hq * d:(Hq + Hkv) * d], qkv[:, (Hq + Hkv) * d:]
o = torch.empty(T, Hq * d, device=DEV, dtype=torch.bfloat16)
cu = torch.tensor([0, T], device=DEV, dtype=torch.int32)
tr = torch.zeros(12, 256, dtype=torch.int64, device=DEV)
run = lambda: lib.prefill_attn(q, k, v, o, cu, 1, T, Hq, Hkv, d, 1 / math.sqrt(d), max_ctas=148)
run(); torch.cuda.synchronize()
lib.load().hp_set_trace(0, tr.data_ptr())
run(); torch.cuda.synchronize()
lib.load().hp_set_trace(0, None)
t = tr.cpu()
base = int(t[0, 0])
for i in range(40, 60):
    a = [int(t[r, i]) - base for r in range(12)]
    # softmax tile A: wait_start, wait_end, ld_done, p_done ; tile B same ; mma: pA wait start/end, pB start/end
    print(f"j={i:3d} A: wait {a[1]-a[0]:6d} ld {a[2]-a[1]:5d} sm {a[3]-a[2]:6d} | B: wait {a[5]-a[4]:6d} ld {a[6]-a[5]:5d} sm {a[7]-a[6]:6d} "
          f"| mma pA wait {a[9]-a[8]:6d} pB wait {a[11]-a[10]:6d} | A.s_ready@{a[1]:9d} A.p@{a[3]:9d} B.s_ready@{a[5]:9d} B.p@{a[7]:9d}")
