"""Full-size parity for the large BASELINE configs (4a, 4b, 4c: 10^8-vertex
tori and chain; 5: RMAT scale 25, ~1.05e9 slots) -- part of the default
``pytest -m gpu`` run.

Each CSR is built on the device (workloads.make_device: the same PCG64 draws
and candidate order as the host generators, symmetrised on the GPU) and its
sha256 is asserted equal to the digest of the CSR the reference consumed
(tests/golden/configs.json, written by tests/golden/make_golden.py from the
reference run).  The pipeline's label / head / is_ap / edge_label are then
compared by sha256 with the REFERENCE's own outputs on that CSR
(fastbcc.fast_bcc, bcc.py:147-196, canonicalised per SURVEY §8(c)), and the
counts exactly.  These sizes exercise paths the small graphs cannot: the
multi-launch tile table (> 16384 tiles, n > 33.5 M), 4-5 ruling-set levels,
RMAT hubs and super-heavy rows, 10^8-long tours.

``FBCC_LARGE=1`` additionally re-runs the golden-pinned C oracle on the same
CSR and compares every array element-wise (minutes per config).
"""

import hashlib
import json
import os
import time

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(memoryview(np.ascontiguousarray(a)).cast("B"))
    return h.hexdigest()


@pytest.mark.parametrize("name", ["4c", "4a", "4b", "5"])
def test_large_config(name):
    sel = os.environ.get("FBCC_LARGE_CONFIGS")
    if sel and name not in sel.split(","):
        pytest.skip("not selected by FBCC_LARGE_CONFIGS")
    import workloads
    from paper_2301_01356_b200.bcc import Plan

    meta = json.loads((GOLDEN / "configs.json").read_text())[name]
    t0 = time.time()
    off, adj = workloads.make_device(name)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    offsets = off.cpu().numpy()
    edges = adj.cpu().numpy().view(np.uint32)
    assert offsets.size - 1 == meta["n"] and edges.size == meta["m"]
    assert _sha(offsets.astype(np.int64, copy=False), edges) == meta["csr_sha256"], "CSR differs from the reference's"

    plan = Plan(off, adj, timing=True)
    plan.run()  # warm
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    st = plan.run()
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    res = {k: (v.cpu().numpy() if v is not None else None) for k, v in plan.outputs().items()}
    stage_ms = [round(float(x), 3) for x in st.stage_ms]
    del plan, off, adj
    torch.cuda.empty_cache()

    assert int(st.num_bccs) == meta["num_bccs"]
    assert int(st.num_components) == meta["num_components"]
    assert int(res["is_ap"].sum()) == meta["num_ap"]
    assert res["edge_label"].size == meta["E"]
    assert _sha(res["label"]) == meta["label_sha256"], "label"
    assert _sha(res["head"]) == meta["head_sha256"], "head"
    assert _sha(res["is_ap"]) == meta["is_ap_sha256"], "is_ap"
    assert _sha(res["edge_label"]) == meta["edge_label_sha256"], "edge_label"

    if name == "5":  # the host path at this size too: streamed upload, the rows' first arcs recorded on the
        # device after it, sampled tags with the repair on the streamed forest (plans of n >= 2^22, m >= 8n)
        from paper_2301_01356_b200 import Graph, fast_bcc

        lab = fast_bcc(Graph(offsets.astype(np.int64, copy=False), edges).pin())
        assert lab.num_bccs == meta["num_bccs"] and lab.num_components == meta["num_components"]
        assert _sha(np.asarray(lab.label)) == meta["label_sha256"], "host path: label"
        assert _sha(np.asarray(lab.head)) == meta["head_sha256"], "host path: head"
        assert _sha(np.asarray(lab.edge_label)) == meta["edge_label_sha256"], "host path: edge_label"
        assert _sha(np.asarray(lab.is_ap).astype(np.uint8)) == meta["is_ap_sha256"], "host path: is_ap"
        del lab
        torch.cuda.empty_cache()

    oracle_s = None
    if os.environ.get("FBCC_LARGE") == "1":  # element-wise against the C oracle too
        import oracle

        oracle.build()
        t1 = time.time()
        ref = oracle.fast_bcc(offsets, edges)
        oracle_s = time.time() - t1
        for k in ("label", "head", "edge_label", "is_ap"):
            assert np.array_equal(res[k], ref[k]), k
    E = edges.size // 2
    line = {"config": name, "n": offsets.size - 1, "E": E, "gpu_ms": ms, "stage_ms": stage_ms,
            "edges_per_s": E / (ms / 1e3), "num_bccs": int(st.num_bccs),
            "num_components": int(st.num_components), "match_reference_digests": True,
            "oracle_s": oracle_s, "gen_s": gen_s}
    print("LARGE " + json.dumps(line), flush=True)  # only after every assert passed
