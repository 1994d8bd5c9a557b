"""Per-CTA windows of one k_fa2 launch (hp_set_trace kind 2: {smid, start_ns,
end_ns} after the programmatic-dependency wait) beside its CUDA-event time:
launch latency, start skew across CTAs, and the spread of CTA finish times.

    python tools/fa_ctas.py [T sms ...]
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_19516_b200.device import lib

DEV = torch.device("cuda", 0)
d, Hq, Hkv = 128, 32, 8
args = [int(a) for a in sys.argv[1:]] or [1024, 124, 4096, 140, 16384, 140]
for T, sms in zip(args[::2], args[1::2]):
    qkv = torch.randn(T, (Hq + 2 * Hkv) * d, device=DEV).to(torch.bfloat16)
    q, k, v = qkv[:, :Hq * d], qkv[:, Hq * d:(Hq + Hkv) * d], qkv[:, (Hq + Hkv) * d:]
    o = torch.empty(T, Hq * d, device=DEV, dtype=torch.bfloat16)
    cu = torch.tensor([0, T], device=DEV, dtype=torch.int32)
    run = lambda: lib.prefill_attn(q, k, v, o, cu, 1, T, Hq, Hkv, d, 1 / math.sqrt(d), max_ctas=sms)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    buf = torch.zeros(sms, 3, dtype=torch.int64, device=DEV)
    torch.cuda._sleep(200_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    lib.load().hp_set_trace(2, buf.data_ptr())
    run()
    b.record()
    torch.cuda.synchronize()
    t = buf.cpu().double()
    st, en = t[:, 1], t[:, 2]
    s0 = st.min()
    dur = (en - st) / 1e3
    print(f"T={T} sms={sms}: event {a.elapsed_time(b) * 1e3:.1f} us | CTA start skew {(st.max() - s0) / 1e3:.1f} us "
          f"| first start -> last end {(en.max() - s0) / 1e3:.1f} us | CTA busy min/median/max "
          f"{dur.min():.1f}/{dur.median():.1f}/{dur.max():.1f} us", flush=True)
