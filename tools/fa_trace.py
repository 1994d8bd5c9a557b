"""clock64 trace of k_fa2's CTA 0 (softmax warp of each tile + MMA waits)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_19516_b200.device import lib
DEV = torch.device("cuda", 0)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
SMS = int(sys.argv[2]) if len(sys.argv) > 2 else 148
d, Hq, Hkv = 128, 32, 8
qkv = torch.randn(T, (Hq + 2 * Hkv) * d, device=DEV).to(torch.bfloat16)
q, k, v = qkv[:, :Hq * d], qkv[:, Hq * d:(Hq + Hkv) * d], qkv[:, (Hq + Hkv) * d:]
o = torch.empty(T, Hq * d, device=DEV, dtype=torch.bfloat16)
cu = torch.tensor([0, T], device=DEV, dtype=torch.int32)
tr = torch.zeros(18, 256, dtype=torch.int64, device=DEV)
run = lambda: lib.prefill_attn(q, k, v, o, cu, 1, T, Hq, Hkv, d, 1 / math.sqrt(d), max_ctas=SMS)
run(); torch.cuda.synchronize()
lib.load().hp_set_trace(0, tr.data_ptr())
ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ea.record()
run()
eb.record()
torch.cuda.synchronize()
lib.load().hp_set_trace(0, None)
import pynvml
pynvml.nvmlInit()
print(f"traced launch: {ea.elapsed_time(eb) * 1e3:.1f} us (events); SM clock now "
      f"{pynvml.nvmlDeviceGetClockInfo(pynvml.nvmlDeviceGetHandleByIndex(0), pynvml.NVML_CLOCK_SM)} MHz")
t = tr.cpu()
base = int(t[0, 0])
for i in range(40, 60):
    a = [int(t[r, i]) - base for r in range(12)]
    # softmax tile A: wait_start, wait_end, ld_done, p_done ; tile B same ; mma: pA wait start/end, pB start/end
    print(f"j={i:3d} A: wait {a[1]-a[0]:6d} ld {a[2]-a[1]:5d} sm {a[3]-a[2]:6d} | B: wait {a[5]-a[4]:6d} ld {a[6]-a[5]:5d} sm {a[7]-a[6]:6d} "
          f"| mma pA wait {a[9]-a[8]:6d} pB wait {a[11]-a[10]:6d} | A.s_ready@{a[1]:9d} A.p@{a[3]:9d} B.s_ready@{a[5]:9d} B.p@{a[7]:9d}")

# per unit (CTA 0): MMA warp waiting for Q, unit span on the tensor core
# (Q ready -> last commit), softmax-A epilogue wait and duration
print("unit  q_wait  mma_span  epi_wait(o_full)  epi  gap_to_next_q")
nu = int((t[12] > 0).sum())
cyc = int(max(t[15, nu - 1], t[13, nu - 1]) - t[16, 0])
print(f"CTA 0: {nu} units, {cyc} cycles from first Q wait to last epilogue = {cyc / 1965:.1f} us at 1965 MHz")
for u in range(256):
    if int(t[12, u]) == 0:
        break
    q_wait = int(t[12, u] - t[16, u])
    span = int(t[13, u] - t[12, u])
    ew = int(t[14, u] - t[17, u]) if int(t[17, u]) else -1
    ep = int(t[15, u] - t[14, u]) if int(t[14, u]) else -1
    nxt = int(t[16, u + 1] - t[13, u]) if u + 1 < 256 and int(t[16, u + 1]) else -1
    print(f"{u:4d} {q_wait:7d} {span:9d} {ew:9d} {ep:6d} {nxt:8d}")
