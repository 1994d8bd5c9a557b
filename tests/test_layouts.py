"""Device memory layouts: the paged-KV page layout helpers (CPU) and the
tiled weight layout (GPU kernel vs a torch restatement)."""

import pytest
import torch

from paper_2504_19516_b200.device import lib


def kv_index(blk, h, off, j, Hkv, page, d):
    """Element index of (block, kv head, token offset, dim) in the device page
    layout -- the formula of k_rope_kv_write (layer_ops.cu)."""
    return ((((blk * Hkv + h) * (page // 64) + off // 64) * (d // 64) + j // 64) * 4096
            + (off & 63) * 64 + ((((j & 63) >> 3) ^ (off & 7)) << 3) + (j & 7))


@pytest.mark.parametrize("d,P", [(64, 64), (128, 64), (128, 192)])
def test_kv_pack_matches_kernel_index_and_roundtrips(d, P):
    nb, H = 3, 2
    x = torch.arange(nb * H * P * d, dtype=torch.float32).view(nb, H, P, d)
    packed = kv_pack_flat = lib.kv_pack(x).reshape(-1)
    g = torch.Generator().manual_seed(0)
    for _ in range(500):
        b, h, o, j = (int(torch.randint(0, n, (1,), generator=g)) for n in (nb, H, P, d))
        assert packed[kv_index(b, h, o, j, H, P, d)] == x[b, h, o, j]
    assert torch.equal(lib.kv_unpack(lib.kv_pack(x)), x)
    del kv_pack_flat


def tile_ref(w):
    N, K = w.shape
    # [N/128][K/128][2][128][64] == [N/128][K/64][128][64]: 128-row x 64-col
    # SW128 boxes, two per contiguous 32 KB [128 x 128] tile
    t = w.view(N // 128, 128, K // 64, 8, 8).permute(0, 2, 1, 3, 4)  # [nb, kb, r, c, e]
    r = torch.arange(128, device=w.device)
    c = torch.arange(8, device=w.device)
    src = (c[None, :] ^ (r[:, None] & 7))[None, None, :, :, None].expand(N // 128, K // 64, 128, 8, 8)
    return torch.gather(t, 3, src).contiguous().view(N, K)


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_tile_weight_kernel_matches_reference_permutation():
    w = torch.randn(384, 640, device="cuda").to(torch.bfloat16)
    assert torch.equal(lib.tile_weight(w), tile_ref(w))
