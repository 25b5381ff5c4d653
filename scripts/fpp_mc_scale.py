#!/usr/bin/env python3
"""Monte-Carlo FPP oracle at scale: an 8 GiB filter (2^28 blocks) at the
BASELINE densities, 10^9 probes each, against the series sbbf_fpp(a)."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_01719_b200.fppsim import sbbf_fpp, sbbf_fpp_mc  # noqa: E402

for a in (24.4140625, 30.517578125, 23.84185791015625, 29.802322387695312):
    t0 = time.perf_counter()
    got = sbbf_fpp_mc(a, 1 << 28, 1_000_000_000, 2026)
    dt = time.perf_counter() - t0
    s = sbbf_fpp(a)
    se = math.sqrt(s * (1 - s) / 1e9)
    print(f"a={a:.6f} blocks=2^28 keys~{a * 2**28:.3e} trials=1e9  mc={got:.7f} series={s:.7f} "
          f"z={(got - s) / se:+.2f}  wall={dt:.2f}s")
