"""tcgen05.mma throughput (M=128, K=16, bf16) by N and operand form; issued
back to back from a converged warp into `chains` accumulators (negative
chains: A operand from TMEM, the TS form used for P.V in k_fa2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_19516_b200.device import lib
out = torch.zeros(148 * 2, dtype=torch.int64, device="cuda")
for bn in (32, 64, 128, 256):
    for chains in (1, 2, -1, -2):
        if abs(chains) * bn > 256:
            continue
        for ctas in (1, 148):
            n = 8192
            lib.check(lib.load().hp_umma_rate(n, bn, chains, ctas, out.data_ptr(), 0))
            torch.cuda.synchronize()
            o = out[: 2 * ctas].view(-1, 2).float().mean(0)
            print(f"N={bn:3d} {'TS' if chains < 0 else 'SS'} chains={abs(chains)} ctas={ctas:3d}: issue {o[0].item() / n:6.1f} "
                  f"complete {o[1].item() / n:6.1f} cyc/mma -> {128 * bn * 16 / (o[1].item() / n):7.0f} MAC/cyc/SM "
                  f"({100 * 128 * bn * 16 / (o[1].item() / n) / 4096:.0f}% of 4096)", flush=True)
