"""Per-CTA timeline of the decode swap-AB GEMM (globaltimer, ns) vs the
CUDA-event span: where the fixed per-launch cost goes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_19516_b200.device import lib
DEV = torch.device("cuda", 0)
for (N, K) in ((4096, 4096), (6144, 4096), (4096, 14336), (28672, 4096)):
    for sms in (148, 32):
        T = 32
        x = torch.randn(T, K, device=DEV).to(torch.bfloat16)
        w = lib.tile_weight((torch.randn(N, K, device=DEV) * 0.02).to(torch.bfloat16))
        y = torch.empty(T, N, device=DEV, dtype=torch.bfloat16)
        ws = torch.empty(lib.gemm_swap_ws_bytes(T, N, K, sms) // 4, device=DEV)
        cnt = torch.zeros(N // 128, device=DEV, dtype=torch.int32)
        tr = torch.zeros(sms, 10, dtype=torch.int64, device=DEV)
        fl = torch.ones(64 << 20, device=DEV)
        for it in range(3):
            fl.sum()
            torch.cuda._sleep(100_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if it == 2:
                lib.load().hp_set_trace(1, tr.data_ptr())
            a.record()
            lib.gemm_swap(x, w, y, ws, cnt, lib.EPI_STORE, max_ctas=sms)
            b.record()
            lib.load().hp_set_trace(1, None)
        torch.cuda.synchronize()
        t = tr.cpu().double()
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3
        sp = t[t[:, 6] > 0]
        if len(sp):
            r2 = (sp - t0) / 1e3
            last = r2[r2[:, 8] > 0]
            print(f"   split tiles: partial written {r2[:, 6].median():.1f}/{r2[:, 6].max():.1f} | counted "
                  f"{r2[:, 7].median():.1f}/{r2[:, 7].max():.1f} | last arrivers {len(last)}: summed "
                  f"{last[:, 8].median():.1f}/{last[:, 8].max():.1f} emitted {last[:, 9].median():.1f}/"
                  f"{last[:, 9].max():.1f} | MMA done of those {last[:, 3].median():.1f}/{last[:, 3].max():.1f}",
                  flush=True)
        print(f"N={N:5d} K={K:5d} sms={sms:3d} event {a.elapsed_time(b)*1e3:6.1f} us | entry [{rel[:,0].min():.1f},{rel[:,0].max():.1f}] "
              f"prologue {(rel[:,1]-rel[:,0]).mean():.1f} | producer done {rel[:,2].median():.1f}/{rel[:,2].max():.1f} "
              f"| mma done {rel[:,3].median():.1f}/{rel[:,3].max():.1f} | epi done {rel[:,4].median():.1f}/{rel[:,4].max():.1f} | exit max {rel[:,5].max():.1f}", flush=True)
