import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_19516_b200.device import lib
out = torch.zeros(148 * 2, dtype=torch.int64, device="cuda")
for bn in (32, 128, 256):
    for chains in (1, 2, 4):
        if chains * bn > 512:
            continue
        for ctas in (1, 148):
            lib.check(lib.load().hp_umma_rate(4096, bn, chains, ctas, out.data_ptr(), 0))
            torch.cuda.synchronize()
            o = out[: 2 * ctas].view(-1, 2).float().mean(0)
            print(f"N={bn:3d} chains={chains} ctas={ctas:3d}: issue {o[0].item() / 4096:6.1f} cyc/mma, "
                  f"complete {o[1].item() / 4096:6.1f} cyc/mma  -> {128 * bn * 16 / (o[1].item() / 4096):7.0f} MAC/cyc/SM", flush=True)
