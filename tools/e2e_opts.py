"""Median end-to-end fast_bcc time on a pinned host graph (fbcc_run_host) under
option variants.  Usage: python tools/e2e_opts.py CONFIG name=v[,name=v] ..."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import workloads
    from paper_2301_01356_b200 import Graph, _lib, fast_bcc

    cfg = sys.argv[1]
    variants = sys.argv[2:] or [""]
    g = workloads.make(cfg)
    gp = Graph(g.offsets, g.edges).pin()
    dev = torch.device("cuda", 0)
    defaults = {k: _lib.get_option(k) for k in _lib.OPTIONS}
    ref = None
    for var in variants:
        for k, v in defaults.items():
            _lib.set_option(k, v)
        for kv in filter(None, var.split(",")):
            k, v = kv.split("=")
            _lib.set_option(k, int(v))
        for _ in range(3):
            lab = fast_bcc(gp, device=dev)
        ts = []
        for _ in range(20):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            lab = fast_bcc(gp, device=dev)
            ts.append(time.perf_counter() - t0)
        sig = (lab.num_bccs, int(np.asarray(lab.edge_label).astype(np.int64).sum()), int(lab.label.sum()))
        ref = ref or sig
        print(f"config {cfg} [{var or 'defaults'}] e2e median {1e3 * np.median(ts):.3f} ms  min {1e3 * min(ts):.3f}"
              f"  stages {[round(x, 3) for x in lab.timings.stage_ms]}"
              f"  same={sig == ref}")


if __name__ == "__main__":
    main()
