"""clock64 trace of k_decode_attn's CTA 0 (build with -DHP_DA_TRACE via
tools/build_variant.sh and point HP_LIB at it): per consumer tile the cycles
spent waiting for K, in QK, softmax, waiting for V, in PV; per producer the
empty-slot waits.

    HP_LIB=exp_builds/datrace/libb200hot.so python tools/da_trace.py [sms]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_19516_b200.device import lib  # noqa: E402

so = lib.load(os.environ["HP_LIB"])
sys.path.insert(0, "tools")
from dattn_shapes import run  # noqa: E402

sms = int(sys.argv[1]) if len(sys.argv) > 1 else 8
gbs, us, nb = run(32, 8, 128, 32, 2048, sms=sms, reps=1)
print(f"sms {sms}: {us:.1f} us {gbs / sms:.1f} GB/s/SM")
full = np.zeros(12 * 64 * 6 + 64 * 4, dtype=np.int64)
so.hp_da_trace_read.argtypes = [ctypes.c_void_p]
assert so.hp_da_trace_read(full.ctypes.data) == 0
buf = full[:12 * 64 * 6].reshape(12, 64, 6)
ut = full[12 * 64 * 6:].reshape(64, 4)
t0 = buf[buf > 0].min()
print("units (consumer warp 0, CTA 0): cycles  [tiles, merge, gap-to-next]")
for k in range(min(63, int((ut[:, 0] > 0).sum()) - 1)):
    print(f"  unit {k:2d}: tiles {ut[k, 1] - ut[k, 0]:6d} merge {ut[k, 3] - ut[k, 1]:6d} gap {ut[k + 1, 0] - ut[k, 3]:6d}")
for w in range(8):
    rows = buf[w]
    print(f"consumer {w}: tile  wait_K  QK  softmax  wait_V  PV  (cycles; start rel)")
    for i in range(0, 24):
        r = rows[i]
        if r[0] == 0:
            break
        print(f"  {i:3d} start {r[0] - t0:8d} waitK {r[1] - r[0]:6d} qk {r[2] - r[1]:6d} soft {r[3] - r[2]:6d} "
              f"waitV {r[4] - r[3]:6d} pv {r[5] - r[4]:6d} total {r[5] - r[0]:6d}")
for pw in range(4):
    rows = buf[8 + pw]
    w = [int(r[1] - r[0]) for r in rows if r[0]]
    st = [int(r[0]) for r in rows if r[0]]
    per = [b - a for a, b in zip(st, st[1:])]
    print(f"producer {pw}: empty waits (cycles): {w[:16]}")
    print(f"producer {pw}: issue period (cycles): {per[:16]}")
    seg = [(int(r[0] - r[5]), int(r[2] - r[1]), int(r[3] - r[2]), int(r[4] - r[3])) for r in rows if r[0]]
    print(f"producer {pw}: (select, expect_tx, bulk copy, tag) cycles: {seg[:8]}")
