"""HBM streaming probes on green-context partitions (one tool, several sweeps).

    python tools/membw.py sweep     # GB/s vs SM count, LDG (method 0) and bulk copy (1)
    python tools/membw.py chunks    # per-SM bulk-copy GB/s vs chunk size, issuing warps, wait mode
    python tools/membw.py lanes     # issuing lanes inside one warp vs issuing warps (16 SMs)
    python tools/membw.py blocked   # blocked vs interleaved chunk assignment (32 SMs)
    python tools/membw.py pipe      # producer-warp pipeline (hp_membw_pipe) vs producers
    python tools/membw.py 2d        # 1-D bulk vs 2-D TMA boxes (hp_membw2d)

Method codes of `hp_membw` (membw.cu): 0 = LDG, 1 = bulk copy, 10 + k = bulk
copies of 4 KB << k, + 8·log2(warps) issuing warps, + 64·spin (spin wait),
+ 64·lanes (lanes of one warp issuing), + 1024 (blocked assignment).
Results feed profiles/calib_b200/bandwidth.json and DESIGN §4.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_19516_b200.device import lib
from paper_2504_19516_b200.device.partition import DECODE, PartitionPool

GIB = 1 << 30


def timed(st, fn, reps=3):
    """Best-of-(reps-1) device time of fn() on the partition's stream (s)."""
    ts = []
    with torch.cuda.stream(st.torch_stream):
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(100000)
            a.record()
            fn()
            b.record()
            ts.append((a, b))
    torch.cuda.synchronize()
    return min(x.elapsed_time(y) for x, y in ts[1:]) * 1e-3


def per_sm(st, buf, out, method, ctas=None):
    t = timed(st, lambda: lib.membw(buf, ctas or st.sms, method, out, stream=st.torch_stream))
    return buf.numel() * buf.element_size() / t / 1e9 / st.sms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["sweep", "chunks", "lanes", "blocked", "pipe", "2d"])
    a = ap.parse_args()
    pool = PartitionPool(0)
    out = torch.zeros(4, device="cuda")
    buf = torch.ones(GIB // 4, dtype=torch.float32, device="cuda")
    nbytes = GIB

    if a.mode == "sweep":
        for method in (0, 1):
            for sms in [8, 16, 24, 32, 40, 48, 56, 64, 80, 96, 112, 128, 144, pool.n]:
                st = pool.phase(DECODE, sms)
                v = per_sm(st, buf, out, method, ctas=st.sms * (4 if method == 0 else 1))
                print(f"method {method} sms {st.sms:3d}: {v * st.sms:8.1f} GB/s  ({v:6.1f} GB/s/SM)", flush=True)
    elif a.mode == "chunks":
        for sms in (8, 32):
            st = pool.phase(DECODE, sms)
            for spin in (0, 1):
                for wl in (0, 2):
                    line = f"sms {st.sms:3d} spin {spin} warps {1 << wl}:"
                    for k in range(5):
                        if (192 * 1024) // (4096 << k) >= (1 << wl):
                            line += f"  {4 << k:2d}KB {per_sm(st, buf, out, 10 + k + 8 * wl + 64 * spin):6.1f}"
                    print(line, flush=True)
    elif a.mode == "lanes":
        st = pool.phase(DECODE, 16)
        for lanes in (2, 4, 8):
            line = f"sms 16 lanes-in-one-warp {lanes}:"
            for k in range(4):
                if (192 * 1024) // (4096 << k) >= lanes:
                    line += f"  {4 << k:2d}KB {per_sm(st, buf, out, 10 + k + 64 * lanes):6.1f}"
            print(line, flush=True)
        for wl in (1, 3):
            line = f"sms 16 warps {1 << wl}:"
            for k in range(4):
                if (192 * 1024) // (4096 << k) >= (1 << wl):
                    line += f"  {4 << k:2d}KB {per_sm(st, buf, out, 10 + k + 8 * wl):6.1f}"
            print(line, flush=True)
    elif a.mode == "blocked":
        st = pool.phase(DECODE, 32)
        for blocked in (0, 1):
            for wl in (0, 2):
                line = f"sms 32 blocked {blocked} warps {1 << wl}:"
                for k in (2, 3):
                    line += f"  {4 << k:2d}KB {per_sm(st, buf, out, 10 + k + 8 * wl + 1024 * blocked):6.1f}"
                print(line, flush=True)
    elif a.mode == "pipe":
        st = pool.phase(DECODE, 32)
        h = lib.load()
        for np_ in (1, 2, 4, 8):
            line = f"sms 32 pipe producers {np_}:"
            for kb in (16, 32):
                if 192 // kb >= np_:
                    t = timed(st, lambda: lib.check(h.hp_membw_pipe(buf.data_ptr(), nbytes, st.sms, kb, np_,
                                                                    out.data_ptr(), st.stream)))
                    line += f"  {kb}KB {nbytes / t / 1e9 / st.sms:6.1f}"
            print(line, flush=True)
    else:  # 2d
        del buf
        rows, cols = 131072, 4096  # 1 GiB bf16
        b2 = torch.ones(rows, cols, dtype=torch.bfloat16, device="cuda")
        h = lib.load()
        for sms in (8, 32, 64, 148):
            st = pool.phase(DECODE, sms)
            t1 = timed(st, lambda: h.hp_membw(b2.data_ptr(), nbytes, st.sms, 1, out.data_ptr(), st.stream), 4)
            line = f"sms {st.sms:3d}: bulk1d {nbytes / t1 / 1e9:7.1f} GB/s"
            for br in (32, 64, 128, 256):
                t = timed(st, lambda: lib.check(h.hp_membw2d(b2.data_ptr(), rows, cols, br, st.sms,
                                                             out.data_ptr(), st.stream)), 4)
                line += f" | 2d box{br:3d} {nbytes / t / 1e9:7.1f}"
            # 2-D boxes over a narrow matrix (row pitch 128 B: contiguous boxes)
            t = timed(st, lambda: lib.check(h.hp_membw2d(b2.data_ptr(), rows * cols // 64, 64, 128, st.sms,
                                                         out.data_ptr(), st.stream)), 4)
            line += f" | 2d box128 contiguous {nbytes / t / 1e9:7.1f}"
            print(line, flush=True)


if __name__ == "__main__":
    main()
