"""Per-CTA windows of one k_fa2 launch (hp_set_trace kind 2: {smid, start_ns,
end_ns} after the programmatic-dependency wait) beside its CUDA-event time:
launch latency, start skew across CTAs, and the spread of CTA finish times.

    python tools/fa_ctas.py [T sms ...]
"""
import math
import os
import sys

import numpy as np

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
    # per-CTA work under the kernel's snake order (fa_tc.cu snake_unit /
    # unit2_of): KV steps (both tiles) and units; fit busy = a*steps + b*units
    n_qt = (T + 255) // 256
    units = []
    for u in range(n_qt * Hq):
        q0 = (n_qt - 1 - u // Hq) * 256
        nA = min((q0 + 255) // 128, (T + 127) // 128)
        nB = min((q0 + 383) // 128, (T + 127) // 128) if q0 + 128 < T else 0
        units.append(max(nA, nB))
    steps, nun = np.zeros(sms), np.zeros(sms)
    r = 0
    while r * sms < len(units):
        for b_ in range(sms):
            u = r * sms + ((sms - 1 - b_) if r & 1 else b_)
            if u < len(units):
                steps[b_] += units[u]
                nun[b_] += 1
        r += 1
    busy = dur.numpy()
    A = np.stack([steps, nun], 1)
    (a_, b_u), *_ = np.linalg.lstsq(A, busy, rcond=None)
    resid = busy - A @ np.array([a_, b_u])
    smid = t[:, 0].numpy().astype(int)
    slow = np.argsort(resid)[-5:]
    print(f"   fit: {a_:.3f} us per KV step ({a_ * 1965:.0f} cycles) + {b_u:.2f} us per unit; residual rms "
          f"{resid.std():.2f} us; slowest CTAs (smid, resid us): {[(int(smid[i]), round(float(resid[i]), 1)) for i in slow]}")
    if os.environ.get("FA_CTAS_DETAIL"):
        per = busy / steps
        order = np.argsort(per)
        for i in list(order[:6]) + list(order[-6:]):
            print(f"   cta {i:3d} smid {smid[i]:3d} units {int(nun[i])} steps {int(steps[i])} busy {busy[i]:6.1f} us "
                  f"-> {per[i] * 1965:6.0f} cycles/step")
    print(f"T={T} sms={sms}: event {a.elapsed_time(b) * 1e3:.1f} us | CTA start skew {(st.max() - s0) / 1e3:.1f} us "
          f"| first start -> last end {(en.max() - s0) / 1e3:.1f} us | CTA busy min/median/max "
          f"{dur.min():.1f}/{dur.median():.1f}/{dur.max():.1f} us", flush=True)
