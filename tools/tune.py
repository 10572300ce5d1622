"""Tuning harness (GPU box): per-launch device times of one profiled run of
the pipeline under option variants.  Usage:
    python tools/tune.py --config 2 --variant sample_rounds=2,find_halving=1 ...
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch  # noqa: F401

    import workloads
    from paper_2301_01356_b200 import _lib
    from paper_2301_01356_b200.bcc import run_device

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--variant", action="append", default=[])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--raw", action="store_true")
    ap.add_argument("--scalars", action="store_true", help="print the sampling-round counters")
    ap.add_argument("--plan", type=int, default=0, help="time N unprofiled graph replays instead")
    a = ap.parse_args()
    off, adj = workloads.make_device(a.config)
    defaults = {k: _lib.get_option(k) for k in _lib.OPTIONS}
    for var in (a.variant or [""]):
        for k, v in defaults.items():
            _lib.set_option(k, v)
        for kv in filter(None, var.split(",")):
            k, v = kv.split("=")
            _lib.set_option(k, int(v))
        if a.plan:  # unprofiled CUDA-graph replays, L2 flushed before each (as bench.py)
            import torch

            from paper_2301_01356_b200.bcc import Plan

            pl = Plan(off, adj)
            flush = torch.empty(256 << 20, dtype=torch.uint8, device=off.device)
            for _ in range(3):
                pl.run()
            ts = []
            for _ in range(a.plan):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                pl.launch()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            print(f"== variant [{var or 'defaults'}] plan median {np.median(ts):.4f} ms  min {min(ts):.4f} ms")
            del pl
            continue
        run_device(off, adj)  # warm
        if a.scalars:  # device counters at the head of the workspace (common.cuh Scalars)
            from paper_2301_01356_b200 import bcc as _bcc

            ws = next(iter(_bcc._WS.values()))
            sc = ws[:4 * 64].view(torch.int32).cpu().numpy()
            print(f"   ncomp {sc[0]} giant {sc[1]} nbccs {sc[2]} err {sc[3]} E {sc[4]}")
            print(f"   S1 roots after rounds {sc[5:13].tolist()} hooks {sc[21:29].tolist()}")
            print(f"   S5 roots after rounds {sc[13:21].tolist()} hooks {sc[29:37].tolist()} heavy {sc[37:39].tolist()}")
        rows = []
        for _ in range(a.reps):
            res, st = run_device(off, adj, profile=True)
            rows.append([(_lib.kernel_name(st.prof_kind[i]), st.prof_ms[i]) for i in range(st.nprof)])
            tot = st.total_ms
        seq = [(rows[0][i][0], np.median([r[i][1] for r in rows])) for i in range(len(rows[0]))]
        print(f"== variant [{var or 'defaults'}] total {tot:.3f} ms  stages {[round(x, 3) for x in st.stage_ms]}"
              f" bccs {st.num_bccs}")
        if a.raw:
            print("  " + "  ".join(f"{k}:{v * 1e3:.0f}" for k, v in seq))
        agg = {}
        for k, v in seq:
            agg[k] = agg.get(k, 0) + v
        print("  " + "  ".join(f"{k}:{v * 1e3:.0f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:12]))


if __name__ == "__main__":
    main()
