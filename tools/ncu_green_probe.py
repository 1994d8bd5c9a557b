"""Which green-context setups can ncu profile?  argv[1] = number of
partitions created before the launch (1 or 18)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_19516_b200.device import lib  # noqa: E402

n = int(sys.argv[1])
parts = [lib.Partition(8 * (i + 1)) for i in range(n)]
p = parts[0]
st = p.stream(1)
x = torch.randn(64, 4096, dtype=torch.bfloat16, device="cuda")
w = torch.ones(4096, dtype=torch.bfloat16, device="cuda")
y = torch.empty_like(x)
lib.rmsnorm(x, w, y, 1e-5, 8)
lib.rmsnorm(x, w, y, 1e-5, p.decode_sms, st)
st.synchronize()
print("ok", n)
