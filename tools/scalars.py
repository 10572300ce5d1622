"""Dump the device Scalars block after one plan run (debug aid).
Usage: python tools/scalars.py --config 5"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

FIELDS = ["ncomp", "giant", "nbccs", "err", "num_edges"] + [f"nroots{i}" for i in range(16)] + \
         [f"hooks{i}" for i in range(16)] + ["nheavy0", "nheavy1", "has_hubs", "ticket", "giant_cnt",
                                             "tile_ticket", "eheavy", "nmega0", "nmega1", "emega", "nlisted", "tour_len",
                                             "near0", "near1", "jlist_n0", "jlist_n1", "und_n", "und_work_lo",
                                             "und_work_hi", "und_big"]


def main():
    import torch

    import workloads
    from paper_2301_01356_b200.bcc import Plan

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="5")
    a = ap.parse_args()
    off, adj = workloads.make_device(a.config)
    p = Plan(off, adj)
    p.run()
    v = p.ws[:4 * len(FIELDS)].view(torch.int32).cpu().tolist()
    print({k: x for k, x in zip(FIELDS, v)})


if __name__ == "__main__":
    main()
