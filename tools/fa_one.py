"""One prefill-attention launch (causal, one sequence, Llama-3-8B heads) for
ncu: python tools/fa_one.py T sms"""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_19516_b200.device import lib  # noqa: E402

T, sms = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda", 0)
Hq, Hkv, d = 32, 8, 128
qkv = torch.randn(T, (Hq + 2 * Hkv) * d, device=dev).to(torch.bfloat16)
q, k, v = qkv[:, :Hq * d], qkv[:, Hq * d:(Hq + Hkv) * d], qkv[:, (Hq + Hkv) * d:]
o = torch.empty(T, Hq * d, device=dev, dtype=torch.bfloat16)
cu = torch.tensor([0, T], device=dev, dtype=torch.int32)
for _ in range(2):
    lib.prefill_attn(q, k, v, o, cu, 1, T, Hq, Hkv, d, 1 / math.sqrt(d), max_ctas=sms)
torch.cuda.synchronize()
