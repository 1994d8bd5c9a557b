"""Decode QKV GEMM with RoPE + paged K/V write fused into the swap-AB
epilogue (hp_gemm_swap_qkv_rope) against the two-launch path it replaces
(hp_gemm_swap STORE + hp_rope_kv_write): the same bits in the qkv output and
in every cache element, for d = 64 / 128, pages of 64 / 128, token counts
that do and do not fill the swap tile, single-CTA and CTA-pair walks, split
and unsplit k ranges; and against a torch fp32 restatement of RoPE."""

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2504_19516_b200.device import lib  # noqa: E402
from paper_2504_19516_b200.device.layer import rope_table  # noqa: E402

DEV = torch.device("cuda", 0)


def bf(shape, scale=1.0, gen=None):
    return (torch.randn(*shape, generator=gen, device=DEV) * scale).to(torch.bfloat16)


@pytest.mark.parametrize("T,Hq,Hkv,d,page,ctas", [
    (32, 32, 8, 128, 64, 8), (32, 32, 8, 128, 64, 148), (7, 32, 8, 128, 128, 16), (100, 32, 8, 128, 64, 32),
    (256, 32, 8, 128, 64, 148), (1, 32, 8, 128, 64, 4), (40, 4, 2, 64, 64, 8), (17, 8, 2, 64, 128, 148)])
def test_fused_qkv_rope_matches_two_launch_path(T, Hq, Hkv, d, page, ctas):
    g = torch.Generator(device=DEV)
    g.manual_seed(T * 131 + d + page + ctas)
    K = 4096 if d == 128 else 256
    N = (Hq + 2 * Hkv) * d
    x, w = bf((T, K), gen=g), bf((N, K), 0.05, g)
    wt = lib.tile_weight(w)
    nblk = 4 * ((T + page - 1) // page) + 4
    cs = torch.from_numpy(rope_table(16384, d)).to(DEV)
    pos = torch.randint(0, 16000, (T,), generator=g, device=DEV, dtype=torch.int32)
    slots = torch.randperm(nblk * page, generator=g, device=DEV)[:T].to(torch.int32)
    ws = torch.empty(lib.gemm_swap_ws_bytes(T, N, K, 148) // 4 + 1, device=DEV, dtype=torch.float32)
    cnt = torch.zeros(4096, device=DEV, dtype=torch.int32)
    shape = (nblk, Hkv, page, d)
    k0, v0 = torch.zeros(shape, device=DEV, dtype=torch.bfloat16), torch.zeros(shape, device=DEV, dtype=torch.bfloat16)
    k1, v1 = k0.clone(), v0.clone()
    y0 = torch.empty(T, N, device=DEV, dtype=torch.bfloat16)
    y1 = torch.empty_like(y0)
    lib.gemm_swap(x, wt, y0, ws, cnt, lib.EPI_STORE, max_ctas=ctas)
    lib.rope_kv_write(y0, Hq, Hkv, d, pos, cs, slots, k0, v0, page, max_ctas=ctas)
    lib.gemm_swap_qkv_rope(x, wt, y1, Hq, Hkv, d, pos, cs, slots, k1, v1, page, ws, cnt, max_ctas=ctas)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
    assert torch.equal(k0, k1) and torch.equal(v0, v1)
    # RoPE restated in fp32 torch on the bf16 projection (rotate_half)
    proj = (x.float() @ w.float().T).to(torch.bfloat16).float().view(T, Hq + 2 * Hkv, d)
    c = cs[pos.long()]
    cos, sin = c[:, None, : d // 2], c[:, None, d // 2:]
    lo, hi = proj[..., : d // 2], proj[..., d // 2:]
    rot = torch.cat([lo * cos - hi * sin, hi * cos + lo * sin], -1)
    ref = torch.cat([rot[:, : Hq + Hkv], proj[:, Hq + Hkv:]], 1).reshape(T, N)
    err = (y1.float() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-2
