"""Benchmark: FAST-BCC on one B200 (or N independent replicas under torchrun).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One step = the whole six-stage hot path (forest, rooting, tags, fence,
skeleton connectivity, labelling incl. per-edge labels and articulation
flags) over the largest single-GPU BASELINE.json workload, config 5 (RMAT
scale 25, edge factor 16, seed 0: 33.5 M vertices, 524 M undirected edges,
1.05e9 CSR slots; synthetic -- the paper's graphs are not available
offline).  ``value`` = undirected edges/s with the CSR resident in HBM;
``e2e`` = the same metric through the public API ``fast_bcc(g)`` with the CSR
in pinned host memory and the results copied back every step.  L2 (126 MB)
is flushed by a 256 MiB device write before every timed step.  The other
configs (1, 2, 3, 4a, 4b, 4c) are measured device-only in ``configs``, each
with its outputs checked against the reference's digests.

The input CSR's sha256 is asserted equal to the one the reference consumed
(tests/golden/configs.json) before anything is timed.

``--impl reference`` times the reference algorithm's CPU implementation
(the golden-pinned C port in oracle/, parallel mode, all host threads) on
the same CSR -- the reference itself is Python/numba and cannot travel to
the GPU box.

Multi-GPU: the path does not shard; N ranks run N
replicas, value = N * E * K / max-over-ranks time.  ``--gpus N`` without
torchrun re-launches itself under torch.distributed.run with N ranks.
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
        "w_sample": n * (16 + 8 + 12 + 12 + 8 + 8),  # own record, degree, 3 recorded arcs + 3 gathers, (w1, w2) by tour + by vertex
        "nlow": 16 * n + 8 * n + 4 * n,              # offsets pair, the row's first / last arc, count out
        "tile": 2 * n * 16 + 16 * n,                 # A + P in, partials out
        "fence": n * (16 + 16 + 16 + 4),
        "edge_blocks": csr + E * (4 + 4 + 4) + 12 * n,
        "edge_final": E * (4 + 4 + 4),
    }.get(kind)


# Our arm pins its main thread -- and so every thread CUDA and torch create
# later -- to one core before CUDA starts (the GPU arm's host side is one
# thread issuing work).  On this VM an unpinned process uploads the host-path
# CSR measurably slower: 3.3 ms instead of 2.7 ms per fast_bcc call on config
# 2 (Stage 1, i.e. the H2D, 1.8 ms instead of 1.25 ms; the same as running
# the whole process under `taskset -c <any one cpu>`).  The host CSR build and
# the CPU baseline run before the pin (their OpenMP pool keeps the full
# mask); `--impl reference` is never pinned.
PIN_NOTE = "unpinned"


def _pin_process(local_rank):
    global PIN_NOTE
    if not hasattr(os, "sched_setaffinity"):
        return
    try:
        mask = sorted(os.sched_getaffinity(0))
        cpu = mask[-1 - (local_rank % len(mask))]
        os.sched_setaffinity(0, {cpu})
        PIN_NOTE = f"main thread pinned to cpu {cpu} (of {len(mask)}) before CUDA started"
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


BIG = ("4a", "4b", "4c", "5")
DEFAULT_CONFIG = "5"


def _golden(config):
    return json.loads((ROOT / "tests" / "golden" / "configs.json").read_text())[config]


def _sha(*arrays):
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        h.update(memoryview(np.ascontiguousarray(a)).cast("B"))
    return h.hexdigest()


def host_graph(config):
    """The config's CSR on the host (tools/hostgen.c for the large ones),
    checked against the digest of the CSR the reference consumed."""
    import workloads

    t0 = time.perf_counter()
    g = workloads.make(config)
    gen_s = time.perf_counter() - t0
    if workloads.csr_digest(g) != _golden(config)["csr_sha256"]:
        raise SystemExit(f"config {config}: generated CSR differs from the reference's (digest)")
    return g, gen_s


def cpu_baseline(g, config):
    """The reference algorithm on all host cores (golden-pinned C port,
    parallel mode), on the full config graph: 1 run for the large configs
    (5-30 s of CPU work), else the median of 3 after a warm-up."""
    import oracle

    oracle.build()
    E = g.m // 2
    runs = 1 if config in BIG else 3
    if config not in BIG:
        oracle.fast_bcc(g.offsets, g.edges, parallel=True)  # warm-up
    secs, stage = [], None
    for _ in range(runs):
        t0 = time.perf_counter()
        r = oracle.fast_bcc(g.offsets, g.edges, parallel=True)
        secs.append(time.perf_counter() - t0)
        stage = [float(x) for x in r["seconds"]]
    s = statistics.median(secs)
    return {"value": E / s, "unit": UNIT, "cores": oracle.num_threads(), "kind": "port",
            "sample": f"full config-{config} graph ({E} edges), {'1 run' if runs == 1 else f'median of {runs} runs after 1 warm-up'}, "
                      f"{s:.3f} s/run; C port of the reference path, parallel mode (concurrent union-find, "
                      f"splitter list ranking), all {oracle.num_threads()} host threads",
            "seconds_per_run": s, "stage_seconds": dict(zip(["first_cc", "rooting", "tagging", "last_cc", "labelling"], stage))}


def run_reference(args, rank, world):
    """The reference arm: the reference's algorithm on the host cores (the C
    port in parallel mode; the Python/numba reference cannot travel to the
    GPU box), same config, metric and unit as our arm.  Rank 0 only."""
    if rank != 0:
        return 0
    import oracle

    g, gen_s = host_graph(args.config)
    E = g.m // 2
    oracle.build()
    t0 = time.perf_counter()
    oracle.fast_bcc(g.offsets, g.edges, parallel=True)
    first_s = time.perf_counter() - t0
    # each step is one full run; keep the whole arm within ~10 minutes
    warm = args.warmup
    if first_s * (args.warmup - 1 + args.steps) > 600:
        warm = 1
    for _ in range(warm - 1):
        oracle.fast_bcc(g.offsets, g.edges, parallel=True)
    secs = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.fast_bcc(g.offsets, g.edges, parallel=True)
        secs.append(time.perf_counter() - t0)
    tot = sum(secs)
    value = E * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": warm, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": _config(args, g),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "port",
                         "sample": f"full config-{args.config} graph per step; C port of the reference path, "
                                   f"parallel mode, all {oracle.num_threads()} host threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "input_gen_s": gen_s,
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


def _config(args, g, n=None, m=None):
    import workloads

    n = g.n if g is not None else n
    m = g.m if g is not None else m
    return {"workload": f"config {args.config}: {workloads.CONFIGS[args.config][0]} (seed 0)",
            "n": n, "undirected_edges": m // 2, "directed_slots": m,
            "csr_sha256": _golden(args.config)["csr_sha256"],
            "l2": "flushed between timed steps (256 MiB device write)", "parallelism": "replicas"}


def _timed_plan(p, steps, flush, world, dist, dev, E, collect=None, pipelined=True):
    """K steps, each after an L2 flush, bracketed by CUDA events on the
    launching stream; barrier + synchronize on both sides; max over ranks.
    pipelined: each step enqueues the graph + the D2H copy of its counts and
    the host does not wait per step (the per-kernel profile needs the
    synchronous form: its event nodes are re-recorded by every replay)."""
    import torch

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(steps):
        flush.zero_()
        starts[k].record()
        if pipelined:
            p.launch()
        else:
            st = p.run()
            if collect:
                collect(st)
        ends[k].record()
    torch.cuda.synchronize()
    if pipelined:
        for _ in range(steps):
            st = p.collect()
            if collect:
                collect(st)
    if world > 1:
        dist.barrier()
    tot = float(sum(s.elapsed_time(e) for s, e in zip(starts, ends)))
    return replica_value(tot, world, E, steps, dist, dev)[1]


def other_configs(args, dev, flush):
    """Device-only numbers for the configs other than the headline one: the
    CSR built on the device, min(K, 5) plan replays with the L2 flushed, and
    the outputs compared with the reference's digests."""
    import torch

    import workloads
    from paper_2301_01356_b200.bcc import Plan

    out = {}
    for name in ("1", "2", "3", "4a", "4b", "4c", "5"):
        if name == args.config:
            continue
        try:
            off, adj = workloads.make_device(name, device=dev)
            n, m = off.numel() - 1, adj.numel()
            plan = Plan(off, adj)  # production replay (no event nodes)
            tplan = Plan(off, adj, timing=True)  # + stage-boundary events (they cut PDL edges)
            for _ in range(3):
                st = plan.run()
                tplan.run()
            steps = max(1, min(args.steps, 5))
            stage = np.zeros(6)

            def coll(s):
                nonlocal stage
                stage += np.array(list(s.stage_ms))

            tot = _timed_plan(plan, steps, flush, 1, None, dev, m // 2)
            _timed_plan(tplan, steps, flush, 1, None, dev, m // 2, coll, pipelined=False)
            del tplan
            res = plan.outputs()
            meta = _golden(name)
            match = (int(st.num_bccs) == meta["num_bccs"] and int(st.num_components) == meta["num_components"]
                     and all(_sha(res[k].cpu().numpy()) == meta[k + "_sha256"]
                             for k in ("label", "head", "is_ap", "edge_label")))
            ms = tot / steps
            out[name] = {"workload": workloads.CONFIGS[name][0], "n": n, "undirected_edges": m // 2,
                         "ms_per_step": ms, "value": (m // 2) / (ms / 1e3), "unit": UNIT,
                         "stage_ms_timing_plan": [float(x) for x in stage / steps], "steps": steps,
                         "matches_reference_digests": bool(match)}
            del plan, off, adj, res
            torch.cuda.empty_cache()
        except Exception as e:  # keep the headline line alive
            out[name] = {"error": f"{type(e).__name__}: {e}"}
    return out


def run_ours(args, rank, world, local_rank):
    host = None
    cpu = None
    gen_s = None
    if world == 1:
        # host CSR (+ the CPU baseline on all cores) before this process is
        # pinned to one core and before CUDA starts
        host, gen_s = host_graph(args.config)
        if not args.no_cpu_baseline:
            cpu = cpu_baseline(host, args.config)
    if not args.no_pin:
        _pin_process(local_rank)

    import torch
    import torch.distributed as dist

    import workloads
    from paper_2301_01356_b200 import Graph, fast_bcc
    from paper_2301_01356_b200 import _lib
    from paper_2301_01356_b200.bcc import Plan

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    backend = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        backend = dist.get_backend()
    if host is None:  # replicas: every rank builds its CSR on its own GPU, then keeps a host copy
        t0 = time.perf_counter()
        off, adj = workloads.make_device(args.config, device=dev)
        torch.cuda.synchronize()
        gen_s = time.perf_counter() - t0
        host = Graph(off.cpu().numpy(), adj.cpu().numpy().view(np.uint32))
        if workloads.csr_digest(host) != _golden(args.config)["csr_sha256"]:
            raise SystemExit(f"rank {rank}: generated CSR differs from the reference's (digest)")
    else:
        off = torch.from_numpy(host.offsets).to(dev)
        adj = torch.from_numpy(host.edges.view(np.int32)).to(dev)
    n, m = host.n, host.m
    E = m // 2
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    plan = Plan(off, adj)                 # production: the six stages as one CUDA-graph replay
    pplan = Plan(off, adj, profile=True)  # same graph + an event node after every kernel
    for _ in range(max(args.warmup, 3)):
        stats = plan.run()
        pplan.run()
    torch.cuda.synchronize()
    T = n - int(stats.num_components)
    meta = _golden(args.config)
    res = plan.outputs()
    outputs_match = (int(stats.num_bccs) == meta["num_bccs"] and int(stats.num_components) == meta["num_components"]
                     and all(_sha(res[k].cpu().numpy()) == meta[k + "_sha256"]
                             for k in ("label", "head", "is_ap", "edge_label")))
    del res

    # ---- timed region: device-resident CSR (the headline value) ------------
    launches = [0]
    with ClockSampler(local_rank) as clk:
        total_ms = _timed_plan(plan, args.steps, flush, world, dist, dev, E,
                               lambda st: launches.__setitem__(0, launches[0] + int(st.launches)))
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

    prof_total_ms = _timed_plan(pplan, args.steps, flush, world, dist, dev, E, collect, pipelined=False)
    value = world * E * args.steps / (total_ms / 1e3)
    del pplan

    # ---- e2e: public API, pinned host CSR in, results out -----------------
    gp = Graph(host.offsets, host.edges)
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
    e2e_match = (lab.num_bccs == meta["num_bccs"] and _sha(lab.edge_label) == meta["edge_label_sha256"]
                 and _sha(lab.label) == meta["label_sha256"])
    del lab
    e2e_total = replica_value(sum(e2e_s), world, E, args.steps, dist, dev)[1]
    h2d = (4 if getattr(gp, "_pinned_off32", None) is not None else 8) * (n + 1) + 4 * m  # as uploaded
    d2h = 4 * n + 4 * n + 4 * E + n + 64

    extra = None
    if rank == 0 and world == 1 and not args.no_extra_configs:
        del gp
        extra = other_configs(args, dev, flush)

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
            "vs_baseline": None, "dtype": "int32", "data": "synthetic", "config": _config(args, host),
            "e2e": {"value": world * E * args.steps / e2e_total, "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": 1e3 * e2e_total / args.steps,
                    "rank0_step_ms": {"min": 1e3 * min(e2e_s), "median": 1e3 * statistics.median(e2e_s),
                                      "max": 1e3 * max(e2e_s)},
                    "host_threads": PIN_NOTE, "outputs_match_reference": bool(e2e_match)},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm, "unit": "GB/s",
                         "frac": ach / hbm, "traffic": traffic, "peak_source": src,
                         "alg_bytes_per_launch": b, "gather_bound": gather_bound},
            "stage_roofline": stage_roof,
            "pipeline_roofline": {"alg_bytes": sum_alg, "achieved_gbs": sum_alg / (ms / 1e3) / 1e9,
                                  "frac": sum_alg / (ms / 1e3) / 1e9 / hbm},
            "stage_ms": dict(zip(stage_names, [float(x) for x in stage_ms / args.steps])),
            "kernels": kern,
            "profiled_ms_per_step": prof_total_ms / args.steps,
            "gpu_launches": launches,
            "clocks": clocks,
            "num_bccs": int(stats.num_bccs), "num_components": int(stats.num_components),
            "outputs_match_reference": bool(outputs_match),
            "ranks": world, "backend": backend or "none (one process)",
            "input_gen_s": gen_s,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if extra is not None:
            line["configs"] = extra
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def check_ranks(rank, world, local_rank):
    """--check-ranks: bring up the process group the bench uses (NCCL with a
    GPU, gloo without), all-reduce one value, report the group size."""
    import torch
    import torch.distributed as dist

    if torch.cuda.is_available():
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        t = torch.ones(1, device="cuda")
    else:
        dist.init_process_group("gloo")
        t = torch.ones(1)
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"ranks": world, "backend": dist.get_backend(), "allreduce_sum": float(t.item())}),
              flush=True)
    dist.destroy_process_group()
    return 0


def _relaunch(args):
    """--gpus N outside torchrun: re-run this command as N ranks."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra-configs", action="store_true", help="skip the device-only lines of the other configs")
    ap.add_argument("--no-pin", action="store_true", help="our arm: leave the process unpinned")
    ap.add_argument("--check-ranks", action="store_true", help="only bring up the N-rank process group and report it")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _relaunch(args)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.check_ranks:
        return check_ranks(rank, world, local_rank)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
