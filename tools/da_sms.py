"""Decode attention GB/s when confined to `sms` CTAs (grid = max_ctas),
llama3-8b B=32 ctx 2048.  HP_LIB=<path> loads an alternative build
(e.g. one compiled with -DHP_DA_NOCOMPUTE to time the K/V stream alone).

    python tools/da_sms.py [sms ...]
"""
import math
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_19516_b200.device import lib  # noqa: E402

if os.environ.get("HP_LIB"):
    lib.load(os.environ["HP_LIB"])
sys.path.insert(0, "tools")
from dattn_shapes import run  # noqa: E402

for sms in [int(a) for a in sys.argv[1:]] or [8, 16, 32, 148]:
    gbs, us, nb = run(32, 8, 128, 32, 2048, sms=sms)
    print(f"sms {sms:4d}  {us:8.1f} us  {gbs:7.1f} GB/s  {gbs / sms:6.1f} GB/s/SM", flush=True)
