#!/usr/bin/env python3
"""e2e (host buffers) step of config 2, median of 20, for library A/Bs."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
r = bench.run_e2e(2, 20, torch.device("cuda", 0))
print(f"e2e {r['value']:.3f} Gkeys/s  {r['ms_per_step']:.3f} ms  h2d {r['h2d_gbs_achieved']:.1f} of {r['h2d_gbs_peak_measured']:.1f} GB/s")
