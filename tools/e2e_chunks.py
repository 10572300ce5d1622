"""e2e per call under upload-range counts (stream_chunks), one process.
Usage: python tools/e2e_chunks.py CONFIG c1 c2 ..."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import workloads
    from paper_2301_01356_b200 import Graph, _lib, fast_bcc

    g = workloads.make(sys.argv[1])
    gp = Graph(g.offsets, g.edges).pin()
    for rep in range(2):
        for c in map(int, sys.argv[2:]):
            _lib.set_option("stream_chunks", c)
            for _ in range(3):
                fast_bcc(gp)
            ts = []
            for _ in range(20):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                fast_bcc(gp)
                ts.append(time.perf_counter() - t0)
            print(f"config {sys.argv[1]} chunks {c}: median {1e3 * np.median(ts):.3f} ms min {1e3 * min(ts):.3f}")


if __name__ == "__main__":
    main()
