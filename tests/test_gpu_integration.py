"""The drop-in boundary on the GPU.

* The ctypes stub INTEGRATION.md §1 tells a reference maintainer to add is
  executed verbatim (only its relative import and library path adjusted) on
  a stand-in for the reference ``Graph`` -- a class with exactly the
  reference's ``__slots__ = ("offsets", "edges")`` (graphs.py:43-58) -- and
  must reproduce the reference's outputs.
* ``paper_2301_01356_b200.fast_bcc`` accepts that slotted object too.
* A plan is bound to its buffers, not their contents: refilling the same
  buffers with a same-size graph that has a super-heavy row (> 8192 arcs)
  and replaying gives that graph's answer (the plan used to bake
  a content-dependent skip in).
"""

import re
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = Path(__file__).resolve().parent.parent


class RefGraph:
    """Stand-in for fastbcc.graphs.Graph: same slots, same properties."""

    __slots__ = ("offsets", "edges")

    def __init__(self, offsets, edges):
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.edges = np.ascontiguousarray(edges, dtype=np.uint32)

    @property
    def n(self):
        return self.offsets.size - 1

    @property
    def m(self):
        return self.edges.size


def _stub():
    text = (ROOT / "INTEGRATION.md").read_text()
    code = re.search(r"```python\n(# fastbcc/_b200.py.*?)```", text, re.S).group(1)
    code = code.replace("from .bcc import BccLabeling, StepTimings",
                        "from paper_2301_01356_b200.bcc import BccLabeling, StepTimings")
    code = code.replace('ctypes.CDLL("libfastbcc_b200.so")',
                        f'ctypes.CDLL("{ROOT / "paper_2301_01356_b200" / "libfastbcc_b200.so"}")')
    ns = {}
    exec(compile(code, "INTEGRATION.md#stub", "exec"), ns)
    return ns["fast_bcc"]


def test_integration_stub_on_reference_style_graph(corpus):
    stub = _stub()
    for i, name, g in list(corpus.items())[::7]:
        rg = RefGraph(g.offsets, g.edges)
        lab = stub(rg)
        assert np.array_equal(lab.label, corpus.get(i, "label")), name
        assert np.array_equal(lab.head, corpus.get(i, "head")), name
        assert lab.num_bccs == corpus.get(i, "num_bccs"), name
        assert lab.num_components == corpus.get(i, "num_components"), name
        if rg.n:
            assert lab.timings.total > 0 and list(lab.timings.as_dict()) == [
                "first_cc", "rooting", "tagging", "last_cc", "total"]
    with pytest.raises(ValueError):
        stub(RefGraph(corpus.graph(0).offsets, corpus.graph(0).edges), block=1)


def test_fast_bcc_accepts_reference_style_graph(corpus, config_meta):
    import hashlib

    import workloads
    from paper_2301_01356_b200 import articulation_points, fast_bcc

    for i, name, g in list(corpus.items())[::5]:
        lab = fast_bcc(RefGraph(g.offsets, g.edges))
        assert np.array_equal(lab.label, corpus.get(i, "label")), name
        assert np.array_equal(lab.head, corpus.get(i, "head")), name
        assert np.array_equal(lab.edge_label, corpus.get(i, "edge_label")), name
        assert np.array_equal(articulation_points(lab), np.flatnonzero(corpus.get(i, "is_ap"))), name
    g = workloads.make("1")
    lab = fast_bcc(RefGraph(g.offsets, g.edges))
    meta = config_meta["1"]
    assert hashlib.sha256(lab.edge_label.tobytes()).hexdigest() == meta["edge_label_sha256"]
    with pytest.raises(TypeError):
        fast_bcc(object())


def _chain(n):
    from paper_2301_01356_b200.graphs import symmetrize

    i = np.arange(n - 1)
    return symmetrize(np.column_stack([i, i + 1]), n)


def _star(n):
    from paper_2301_01356_b200.graphs import symmetrize

    i = np.arange(1, n)
    return symmetrize(np.column_stack([np.zeros_like(i), i]), n)


def test_plan_is_content_independent():
    from paper_2301_01356_b200.bcc import Plan

    n = 20000
    a, b = _chain(n), _star(n)  # same n and m; the star's hub row has n-1 > 8192 arcs
    assert a.m == b.m
    off = torch.from_numpy(a.offsets).cuda()
    adj = torch.from_numpy(a.edges.view(np.int32)).cuda()
    for first, second in ((a, b), (b, a)):
        off.copy_(torch.from_numpy(first.offsets))
        adj.copy_(torch.from_numpy(first.edges.view(np.int32)))
        plan = Plan(off, adj)
        st = plan.run()
        assert int(st.num_bccs) == n - 1
        for g, n_ap in ((second, None), (first, None)):
            off.copy_(torch.from_numpy(g.offsets))
            adj.copy_(torch.from_numpy(g.edges.view(np.int32)))
            st = plan.run()
            out = plan.outputs()
            ap = out["is_ap"].cpu().numpy()
            assert int(st.num_bccs) == n - 1 and int(st.num_components) == 1
            if g is b:  # star: every edge its own block, one cut vertex (the hub)
                assert np.flatnonzero(ap).tolist() == [0]
                assert np.array_equal(out["edge_label"].cpu().numpy(), np.arange(n - 1))
            else:  # chain: all inner vertices are cut vertices
                assert int(ap.sum()) == n - 2
        del plan


def test_plan_freezes_options():
    from paper_2301_01356_b200 import _lib
    from paper_2301_01356_b200.bcc import Plan

    g = _chain(50000)
    off = torch.from_numpy(g.offsets).cuda()
    adj = torch.from_numpy(g.edges.view(np.int32)).cuda()
    old = _lib.get_option("s0")
    try:
        plan = Plan(off, adj)
        ws_before = _lib.workspace_bytes(g.n, g.m)
        _lib.set_option("s0", 4)  # a different ruling-set layout for plans created from now on
        assert _lib.workspace_bytes(g.n, g.m) > ws_before
        st = plan.run()  # the existing plan keeps its own snapshot (and workspace size)
        assert int(st.num_bccs) == g.n - 1
        plan2 = Plan(off, adj)
        assert int(plan2.run().num_bccs) == g.n - 1
    finally:
        _lib.set_option("s0", old)
