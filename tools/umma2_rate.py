"""tcgen05.mma.cta_group::2 (M=256 pair MMA) throughput vs the 1-CTA forms."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_19516_b200.device import lib
for bn in (32, 64, 128, 256):
    for pairs in (1, 74):
        n = 8192
        out = torch.zeros(4 * pairs, dtype=torch.int64, device="cuda")
        lib.check(lib.load().hp_umma2_rate(n, bn, pairs, out.data_ptr(), 0), "umma2")
        torch.cuda.synchronize()
        o = out.view(2, -1)[:, 0::2].float().mean(1)  # leader CTAs
        per_sm = 128 * bn * 16 / (o[1].item() / n)   # each SM holds 128 of the 256 rows
        print(f"pair M=256 N={bn:3d} pairs={pairs:3d}: issue {o[0].item() / n:6.1f} complete {o[1].item() / n:6.1f} "
              f"cyc/mma -> {per_sm:7.0f} MAC/cyc/SM ({100 * per_sm / 4096:.0f}% of 4096)", flush=True)
