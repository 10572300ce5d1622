"""Median end-to-end fast_bcc time on a pinned host graph with the library
FBCC_LIB points at (A/B of builds on one box).  Usage: python tools/e2e_ab.py CONFIG"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import workloads
    from paper_2301_01356_b200 import Graph, fast_bcc

    g = workloads.make(sys.argv[1])
    gp = Graph(g.offsets, g.edges).pin()
    for _ in range(5):
        lab = fast_bcc(gp)
    ts = []
    for _ in range(30):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lab = fast_bcc(gp)
        ts.append(time.perf_counter() - t0)
    print(f"config {sys.argv[1]} e2e median {1e3 * np.median(ts):.3f} ms min {1e3 * min(ts):.3f} "
          f"stages {[round(x, 3) for x in lab.timings.stage_ms]} bccs {lab.num_bccs}")


if __name__ == "__main__":
    main()
