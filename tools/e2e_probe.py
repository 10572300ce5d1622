"""Break down fast_bcc's end-to-end time on a host graph (fbcc_run_host):
raw link speeds, the run itself, its per-stage events, and the Python-side
overhead around it."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import workloads
    from paper_2301_01356_b200 import Graph, _lib, fast_bcc
    from paper_2301_01356_b200.bcc import _host_session

    cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
    g = workloads.make(cfg)
    gp = Graph(g.offsets, g.edges).pin()
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

    h2d = 8 * (g.n + 1) + 4 * g.m
    d2h = 9 * g.n + 4 * (g.m // 2)
    x = torch.empty(h2d, dtype=torch.uint8).pin_memory()
    y = torch.empty(h2d, dtype=torch.uint8, device=dev)
    print(f"raw h2d {h2d / 1e6:.1f} MB ms", t(lambda: y.copy_(x, non_blocking=True)))
    print(f"raw d2h {d2h / 1e6:.1f} MB ms", t(lambda: x[:d2h].copy_(y[:d2h], non_blocking=True)))
    r = _host_session(gp, dev)
    print("run_host ms", t(lambda: r.run(gp)))
    st, _, _ = r.run(gp)
    print("run_host stage ms", [round(float(v), 3) for v in st.stage_ms], "total", round(float(st.total_ms), 3))
    print("fast_bcc ms", t(lambda: fast_bcc(gp, device=dev)))
    old = _lib.get_option("stream_chunks")
    for c in (1, 2, 4, 16, 32):
        _lib.set_option("stream_chunks", c)
        print(f"run_host chunks={c} ms", t(lambda: r.run(gp)))
    _lib.set_option("stream_chunks", old)


if __name__ == "__main__":
    main()
