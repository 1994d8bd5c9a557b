"""Per-stage device-vs-oracle errors for one Llama-3-8B prefill layer."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import numerics as O
from paper_2504_19516_b200.device.layer import DeviceLayer, KVCache, LayerWeights, PrefillScratch
from paper_2504_19516_b200.workload import MODEL_PRESETS

T = int(sys.argv[1]) if len(sys.argv) > 1 else 512
m = MODEL_PRESETS["llama3-8b"]
rng = np.random.default_rng(0)
bf = lambda a: O.bf16_round(np.asarray(a, np.float32))  # noqa: E731
h, I, d, Hq, Hkv = m.hidden, m.intermediate, m.head_dim, m.num_heads, m.num_kv_heads
W = O.LayerWeights(bf(rng.normal(0, .02, (m.qkv_out_dim, h))), bf(rng.normal(0, .02, (h, h))),
                   bf(rng.normal(0, .02, (I, h))), bf(rng.normal(0, .02, (I, h))), bf(rng.normal(0, .02, (h, I))),
                   bf(1 + .1 * rng.normal(size=h)), bf(1 + .1 * rng.normal(size=h)))
dev = torch.device("cuda", 0)
lyr = DeviceLayer(m, LayerWeights.from_numpy(dev, W.w_qkv, W.w_o, W.w_gate, W.w_up, W.w_down, W.attn_norm, W.mlp_norm), dev, max_pos=T + 2)
t = lambda a, dt=torch.bfloat16: torch.from_numpy(np.ascontiguousarray(a)).to(dt).to(dev)  # noqa: E731
x = bf(rng.normal(size=(T, h)))
sc = PrefillScratch(m, T, dev)
y = torch.empty(T, h, dtype=torch.bfloat16, device=dev)
cache = KVCache(-(-T // 64), Hkv, d, dev)
lyr.prefill(t(x), y, sc, t(np.array([0, T]), torch.int32), 1, T, t(np.arange(T), torch.int32),
            t(np.arange(T), torch.int32), cache, 148)
torch.cuda.synchronize()
g = lambda a: a.float().cpu().numpy()  # noqa: E731
table = O.rope_table(T + 2, d)
qkv = bf(bf(O.rmsnorm(x, W.attn_norm)) @ W.w_qkv.T)
q = bf(O.apply_rope(qkv[:, :Hq * d].reshape(T, Hq, d), np.arange(T), table))
k = bf(O.apply_rope(qkv[:, Hq * d:(Hq + Hkv) * d].reshape(T, Hkv, d), np.arange(T), table))
v = qkv[:, (Hq + Hkv) * d:].reshape(T, Hkv, d)
a = bf(O.causal_attention(q, k, v, 1 / math.sqrt(d)).reshape(T, -1))
hh = bf(x + a @ W.w_o.T)
n2 = bf(O.rmsnorm(hh, W.mlp_norm))
act = bf(O.silu(n2 @ W.w_gate.T) * (n2 @ W.w_up.T))
yy = bf(hh + act @ W.w_down.T)
dq = g(sc.qkv[:T])


def rep(name, dv, rf):
    diff = np.abs(dv - rf)
    i = np.unravel_index(np.argmax(diff), diff.shape)
    print(f"{name:6s} max|d|={diff.max():.5f} at {i} ref={rf[i]:.5f} dev={dv[i]:.5f}  "
          f"mean|d|={diff.mean():.2e} max|ref|={np.abs(rf).max():.3f}")


rep("q", dq[:, :Hq * d], q.reshape(T, -1))
rep("k", dq[:, Hq * d:(Hq + Hkv) * d], k.reshape(T, -1))
rep("v", dq[:, (Hq + Hkv) * d:], v.reshape(T, -1))
rep("attn", g(sc.attn[:T]), a)
rep("h", g(sc.h[:T]), hh)
rep("act", g(sc.act[:T]), act)
rep("y", g(y), yy)
# isolate: device attention from oracle inputs
