"""Break down fast_bcc's end-to-end time (pinned H2D, graph replay, D2H)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import workloads
    from paper_2301_01356_b200 import Graph, fast_bcc
    from paper_2301_01356_b200.bcc import _session, _to_host

    g = workloads.make("2")
    gp = Graph(g.offsets, g.edges)
    gp._pinned = (torch.from_numpy(g.offsets).pin_memory(), torch.from_numpy(g.edges.view(np.int32)).pin_memory())
    dev = torch.device("cuda", 0)
    for _ in range(3):
        fast_bcc(gp, device=dev)
    torch.cuda.synchronize()

    def t(f, reps=10):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return 1e3 * float(np.median(ts))

    plan = _session(gp, dev)
    print("h2d+session ms", t(lambda: _session(gp, dev)))
    print("plan.run ms", t(lambda: plan.run()))
    res = plan.outputs()
    print("d2h (to_host) ms", t(lambda: _to_host(res, ("label", "head", "edge_label", "is_ap"))))
    print("fast_bcc ms", t(lambda: fast_bcc(gp, device=dev)))
    x = torch.empty(75 << 20, dtype=torch.uint8).pin_memory()
    y = torch.empty(75 << 20, dtype=torch.uint8, device=dev)
    print("raw h2d 75MB ms", t(lambda: y.copy_(x, non_blocking=True)))
    print("raw d2h 75MB ms", t(lambda: x.copy_(y, non_blocking=True)))


if __name__ == "__main__":
    main()
