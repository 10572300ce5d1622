"""Benchmark: FAST-BCC on one B200 (or N independent replicas under torchrun).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One step = the whole six-stage hot path (forest, rooting, tags, fence,
skeleton connectivity, labelling incl. per-edge labels and articulation
flags) over the BASELINE.json headline workload, config 2 (uniform random
graph, n = 2^20, m = 8n, seed 0; synthetic -- the paper's graphs are not
available offline).  ``value`` = undirected edges/s with the CSR resident in
HBM; ``e2e`` = the same metric through the public API ``fast_bcc(g)`` with
the CSR in pinned host memory and the results copied back every step.
L2 (126 MB) is flushed by a 256 MiB device write before every timed step
(the config-2 CSR, 71 MB, would otherwise stay L2-resident).

``--impl reference`` times the reference algorithm's CPU implementation
(the golden-pinned C port in oracle/, all host threads) on the same
workload -- the reference itself is Python/numba and cannot travel to the
GPU box.

Multi-GPU: the path does not shard; N ranks run N
replicas, value = N * E * K / max-over-ranks time.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "undirected edges/sec (full BCC, 1 B200)"
UNIT = "edges/s"


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


# Algorithmic bytes per launch of the main kernels: each
# kernel reads its contract inputs once and writes its outputs once, 4-byte
# ids, gathers counted at element size (no sector amplification).
def alg_bytes(kind, n, m, T, E, K1=0):
    csr = 8 * (n + 1) + 4 * m
    return {
        "hook_min": 16 * n + 4 * n + 4 * n + 8 * n,  # off[v..v+1], adj[off[v]], comp + fe out
        "propose": 16 * n + 4 * n + 8 * n,           # per sampling round
        "compress": 8 * n,
        "link_rows": csr + 4 * n + 8 * T,            # one full connectivity pass over the CSR
        "out_lists": n * (4 + 8) + 2 * n * 4,
        "link_tour": 2 * n * (4 + 4 + 8 + 4),
        "walk0": 2 * n * (4 + 8),                    # read succ, write (segment, offset)
        "rank0": 2 * n * (8 + 4 + 4),
        "positions": n * (16 + 16 + 8 + 4) + 2 * n * 8 * 2,
        "firsts": 16 * n + 4 * n,
        "w_gather": csr + 4 * m + 16 * n + 12 * n,   # first[w] per arc + row record + (w1, w2) + nlow out
        "tile": 2 * n * 16 + 16 * n,                 # A + P in, partials out
        "fence": n * (16 + 16 + 16 + 4),
        "edge_blocks": csr + E * (4 + 4 + 4) + 12 * n,
        "edge_final": E * (4 + 4 + 4),
    }.get(kind)


# Our arm pins its process -- the caller and every thread CUDA and torch
# create later -- to one core before CUDA starts (the GPU arm's host side is
# one thread issuing work).  On this VM an unpinned process uploads the
# host-path CSR measurably slower: 3.3 ms instead of 2.7 ms per fast_bcc call
# on config 2 (Stage 1, i.e. the H2D, 1.8 ms instead of 1.25 ms; the same as
# running the whole process under `taskset -c <any one cpu>`).  The CPU
# baseline then runs in a child with the full mask; `--impl reference` is
# never pinned.
FULL_MASK = None
PIN_NOTE = "unpinned"


def _pin_process(local_rank):
    global FULL_MASK, PIN_NOTE
    if not hasattr(os, "sched_setaffinity"):
        return
    try:
        mask = sorted(os.sched_getaffinity(0))
        cpu = mask[-1 - (local_rank % len(mask))]
        os.sched_setaffinity(0, {cpu})
        FULL_MASK = set(mask)
        PIN_NOTE = f"process pinned to cpu {cpu} (of {len(mask)})"
    except OSError:
        pass


def measured_gather_peak(n, gathers):
    """Streamed-index random-gather rate measured by tools/gather_peak.py for
    the gathered-array size closest to n 4-byte words (and gather count)."""
    import math

    try:
        d = json.loads((ROOT / "profiles" / "r1_gather_peak.json").read_text())
        best = min(d["gather"], key=lambda r: (abs(math.log2(r["elements"]) - math.log2(max(n, 2))),
                                               abs(math.log2(r["gathers"]) - math.log2(max(gathers, 2)))))
        return best["streamed_idx_per_s"], (f"profiles/r1_gather_peak.json: {best['array']}, "
                                            f"{best['gathers']} gathers ({d.get('device', '')})")
    except Exception:
        return None, "unavailable"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, p in zip(names, parts[2:]):
                if p.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(g, config, runs=3):
    """The reference algorithm on the host cores (golden-pinned C port).  When
    this process was pinned to one core for the GPU arm (PIN_NOTE), the port
    runs in a child process with every core of the original mask."""
    if FULL_MASK is not None:
        code = ("import json, sys; sys.path.insert(0, %r); import bench, workloads; "
                "print(json.dumps(bench._cpu_baseline_here(workloads.make(%r), %r, %d)))") % (
                    str(ROOT), str(config), str(config), runs)
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True,
                             preexec_fn=lambda: os.sched_setaffinity(0, FULL_MASK))
        return json.loads(out.stdout.strip().splitlines()[-1])
    return _cpu_baseline_here(g, config, runs)


def _cpu_baseline_here(g, config, runs=3):
    import oracle

    oracle.build()
    E = g.m // 2
    oracle.fast_bcc(g.offsets, g.edges)  # warm-up
    secs = []
    for _ in range(runs):
        t0 = time.perf_counter()
        oracle.fast_bcc(g.offsets, g.edges)
        secs.append(time.perf_counter() - t0)
    s = statistics.median(secs)
    return {"value": E / s, "unit": UNIT, "cores": oracle.num_threads(), "kind": "port",
            "sample": f"full config-{config} graph ({E} edges), median of {runs} runs after 1 warm-up, "
                      f"{s:.3f} s/run", "seconds_per_run": s}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import workloads

    g = workloads.make(args.config)
    E = g.m // 2
    import oracle

    oracle.build()
    for _ in range(args.warmup):
        oracle.fast_bcc(g.offsets, g.edges)
    secs = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.fast_bcc(g.offsets, g.edges)
        secs.append(time.perf_counter() - t0)
    tot = sum(secs)
    value = E * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": _config(args, g),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "port",
                         "sample": f"full config-{args.config} graph per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def replica_value(local_total_ms, world, edges_per_replica, steps, dist=None, device=None):
    """Whole-job throughput of N independent replicas: every rank processed
    ``steps`` copies of the workload; the job time is the MAX over ranks of
    the per-rank device time.  Returns (value edges/s, max_total_ms)."""
    total = float(local_total_ms)
    if world > 1:
        import torch

        t = torch.tensor([total], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    return world * edges_per_replica * steps / (total / 1e3), total


def _config(args, g):
    import workloads

    return {"workload": f"config {args.config}: {workloads.CONFIGS[args.config][0]} (seed 0)",
            "n": g.n, "undirected_edges": g.m // 2, "directed_slots": g.m,
            "l2": "flushed between timed steps (256 MiB device write)", "parallelism": "replicas"}


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import workloads
    from paper_2301_01356_b200 import Graph, fast_bcc
    from paper_2301_01356_b200 import _lib
    from paper_2301_01356_b200.bcc import Plan

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    g = workloads.make(args.config)
    n, m = g.n, g.m
    E = m // 2
    off = torch.from_numpy(g.offsets).to(dev)
    adj = torch.from_numpy(g.edges.view(np.int32)).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    plan = Plan(off, adj)                 # production: the six stages as one CUDA-graph replay
    pplan = Plan(off, adj, profile=True)  # same graph + an event node after every kernel
    for _ in range(max(args.warmup, 3)):
        stats = plan.run()
        pplan.run()
    torch.cuda.synchronize()
    T = n - int(stats.num_components)

    def timed(p, collect, pipelined=False):
        """K steps, each after an L2 flush, bracketed by CUDA events on the
        launching stream; barrier + synchronize on both sides; max over ranks.
        pipelined: each step enqueues the graph + the D2H copy of its counts
        and the host does not wait per step (the per-kernel profile needs the
        synchronous form: its event nodes are re-recorded by every replay)."""
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.zero_()
            starts[k].record()
            if pipelined:
                p.launch()
            else:
                collect(p.run())
            ends[k].record()
        torch.cuda.synchronize()
        if pipelined:
            for _ in range(args.steps):
                collect(p.collect())
        if world > 1:
            dist.barrier()
        tot = float(sum(s.elapsed_time(e) for s, e in zip(starts, ends)))
        return replica_value(tot, world, E, args.steps, dist, dev)[1]

    # ---- timed region: device-resident CSR (the headline value) ------------
    launches = [0]
    with ClockSampler(local_rank) as clk:
        total_ms = timed(plan, lambda st: launches.__setitem__(0, launches[0] + int(st.launches)), pipelined=True)
    launches = launches[0]
    # ---- the same K steps with per-kernel event nodes (roofline evidence) --
    per_kernel = {}
    stage_ms = np.zeros(6)

    def collect(st):
        nonlocal stage_ms
        stage_ms += np.array(list(st.stage_ms))
        for i in range(st.nprof):
            name = _lib.kernel_name(st.prof_kind[i])
            tot, cnt = per_kernel.get(name, (0.0, 0))
            per_kernel[name] = (tot + float(st.prof_ms[i]), cnt + 1)

    prof_total_ms = timed(pplan, collect)
    value = world * E * args.steps / (total_ms / 1e3)

    # ---- e2e: public API, pinned host CSR in, results out -----------------
    gp = Graph(g.offsets, g.edges)
    gp.pin()
    for _ in range(max(args.warmup, 3)):  # >= 2 live result sets before the pinned cache is warm
        lab = fast_bcc(gp, device=dev)
    torch.cuda.synchronize()
    e2e_s = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lab = fast_bcc(gp, device=dev)
        e2e_s.append(time.perf_counter() - t0)
    e2e_total = replica_value(sum(e2e_s), world, E, args.steps, dist, dev)[1]
    h2d = (4 if getattr(gp, "_pinned_off32", None) is not None else 8) * (n + 1) + 4 * m  # as uploaded
    d2h = 4 * n + 4 * n + 4 * E + n + 64

    if rank == 0:
        peaks, src = _peaks()
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        # dominant kernel = the kernel kind with the largest device time per step
        kern = {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps,
                    "ms_per_launch": v[0] / v[1]} for k, v in per_kernel.items()}
        dom = max((k for k in kern if alg_bytes(k, n, m, T, E) is not None), key=lambda k: kern[k]["ms_per_step"])
        b = alg_bytes(dom, n, m, T, E)
        ach = b / (kern[dom]["ms_per_launch"] / 1e3) / 1e9
        traffic = None
        prof = ROOT / "profiles" / "ncu_traffic.json"
        if prof.exists():
            try:
                traffic = json.loads(prof.read_text()).get(f"config{args.config}", {}).get(dom)
            except Exception:
                traffic = None
        # Random 4-byte gathers are bounded by the L1TEX line rate (one 128 B
        # wavefront per cycle per SM) long before HBM: report the kernel's
        # gather rate against the rate measured for the same access pattern
        # on this B200 (tools/gather_peak.py: streamed 16 B index loads, 8
        # random 4-byte gathers per thread, gathered array of the same size).
        gathers = {"w_gather": m, "edge_blocks": E}.get(dom)
        clocks = clk.summary()
        gather_bound = None
        if gathers:
            g_rate = gathers / (kern[dom]["ms_per_launch"] / 1e3)
            g_peak, g_src = measured_gather_peak(n, gathers)
            gather_bound = {"gathers_per_launch": gathers, "achieved_per_s": g_rate, "peak_per_s": g_peak,
                            "frac": g_rate / g_peak if g_peak else None, "peak_source": g_src,
                            "l1tex_model_per_s": 148 * (clocks.get("sm_mhz") or 1965.0) * 1e6}
        sum_alg = 46 * m + 165 * n + 48 * T + 16  # SURVEY §8(d) end-to-end algorithmic bytes
        ms = total_ms / args.steps
        # per-stage roofline (each stage reads its contract
        # inputs and writes its outputs once) over the per-stage event times
        stage_names = ["forest", "rooting", "tags", "fence", "skeleton_cc", "labelling"]
        stage_bytes = [4 * (n + 1) + 4 * m + 4 * n + 8 * T, 8 * T + 16 * (2 * T) + 12 * n,
                       4 * (n + 1) + 12 * m + 40 * n, 40 * n, 4 * (n + 1) + 16 * m + 16 * n,
                       4 * (n + 1) + 14 * m + 37 * n]
        stage_roof = {}
        for nm, b_s, t_s in zip(stage_names, stage_bytes, stage_ms / args.steps):
            gbs = b_s / (float(t_s) / 1e3) / 1e9 if t_s > 0 else None
            stage_roof[nm] = {"alg_bytes": int(b_s), "ms": float(t_s), "achieved_gbs": gbs,
                              "frac": gbs / hbm if gbs else None}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic", "config": _config(args, g),
            "e2e": {"value": world * E * args.steps / e2e_total, "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": 1e3 * e2e_total / args.steps,
                    "rank0_step_ms": {"min": 1e3 * min(e2e_s), "median": 1e3 * statistics.median(e2e_s),
                                      "max": 1e3 * max(e2e_s)},
                    "host_threads": PIN_NOTE},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm, "unit": "GB/s",
                         "frac": ach / hbm, "traffic": traffic, "peak_source": src,
                         "alg_bytes_per_launch": b, "gather_bound": gather_bound},
            "stage_roofline": stage_roof,
            "pipeline_roofline": {"alg_bytes": sum_alg, "achieved_gbs": sum_alg / (ms / 1e3) / 1e9,
                                  "frac": sum_alg / (ms / 1e3) / 1e9 / hbm},
            "stage_ms": dict(zip(["forest", "rooting", "tags", "fence", "skeleton_cc", "labelling"],
                                 [float(x) for x in stage_ms / args.steps])),
            "kernels": kern,
            "profiled_ms_per_step": prof_total_ms / args.steps,
            "gpu_launches": launches,
            "clocks": clocks,
            "num_bccs": int(stats.num_bccs), "num_components": int(stats.num_components),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(g, args.config)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pin", action="store_true", help="our arm: leave the process unpinned")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    if args.impl == "ours" and not args.no_pin:
        _pin_process(int(os.environ.get("LOCAL_RANK", 0)))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
