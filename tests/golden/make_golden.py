"""Generate the golden fixtures by RUNNING THE REFERENCE (this container only).

The reference package (/root/reference/pkg, Python + numba) does not exist on
the GPU box, so its outputs are frozen here as small fixtures and committed:

* ``corpus.npz``  -- the reference test corpus (pkg/tests/conftest.py:46-133:
  26 named shapes + families + the 1,020-graph G(n,p) sweep), each graph's
  CSR, and the reference's outputs on it: connected_components labels and
  forest (connectivity.py:593-611), build_euler_tour on that forest
  (euler_tour.py:361-394), compute_tags (tagging.py:300-304), fence bits of
  skeleton_record (connectivity.py:471-480), fast_bcc label/head/num_bccs/
  num_components (bcc.py:147-196), articulation_points (bcc.py:222-235),
  hopcroft_tarjan block count (baselines.py:178-205) and per-edge labels
  (SURVEY §8(c) rule, asserted equal to tv_skeleton(g).edge_label,
  baselines.py:231-303).
* ``listrank.npz`` -- list_ranking (euler_tour.py:322-358) on seeded random
  multi-list inputs, plus the error cases of test_euler_tour.py:143-162.
* ``config1.npz`` -- full outputs on BASELINE config 1 (torus 300x300 p=0.6).
* ``configs.json`` -- for configs 1-3: CSR digest, counts and sha256 digests
  of label/head/is_ap/edge_label (configs 2-3 are too large to commit).

Usage:  python tests/golden/make_golden.py [--skip-configs]
The reference needs one patch on numba 0.65 (SURVEY §0 finding 1): the
``_any_unranked`` prange reduction fails to compile, so the module global is
rebound to a numpy equivalent before the first call.
"""

import argparse
import hashlib
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent


def import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "numba_ref_cache"))
    sys.path.insert(0, str(REF / "src"))
    sys.path.insert(0, str(REF / "tests"))
    import fastbcc
    import fastbcc.euler_tour as et

    et._any_unranked = lambda r: int((r == -1).any())
    return fastbcc


def canonical_edge_labels(g, label, head):
    """SURVEY §8(c) steps 2-4, vectorised."""
    src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.offsets))
    dst = g.edges.astype(np.int64)
    up = src < dst
    u, v = src[up], dst[up]
    lu, lv = label[u], label[v]
    blk = np.where(lu == lv, lu, np.where(head[lv] == u, lv, lu)).astype(np.int64)
    E = u.size
    if E == 0:
        return np.empty(0, np.int32)
    bmin = np.full(g.n, np.iinfo(np.int64).max, np.int64)
    np.minimum.at(bmin, blk, np.arange(E, dtype=np.int64))
    return bmin[blk].astype(np.int32)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def corpus(fb):
    import conftest

    graphs = conftest.corpus_families() + conftest.corpus_random()
    from fastbcc import baselines, bcc, connectivity, euler_tour, tagging

    names, ns, ms, ks, es = [], [], [], [], []
    cols = {k: [] for k in ("offsets", "edges", "cc_label", "forest", "parent",
                            "first", "last", "w1", "w2", "low", "high", "fence",
                            "label", "head", "is_ap", "edge_label")}
    nbccs, ncomps, ht_nbccs = [], [], []
    for name, g in graphs:
        n = g.n
        res = connectivity.connected_components(g)
        f = euler_tour.build_euler_tour(n, res.forest_edges, res.labels)
        tags = tagging.compute_tags(g, f)
        skel = connectivity.skeleton_record(f.parent, f.first, f.last, tags.low, tags.high)
        lab = bcc.fast_bcc(g)
        ap = np.zeros(n, np.uint8)
        ap[bcc.articulation_points(lab)] = 1
        el = canonical_edge_labels(g, lab.label, lab.head)
        if g.m:
            tv = baselines.tv_skeleton(g).edge_label
            assert np.array_equal(tv.astype(np.int64), el.astype(np.int64)), name
        ht = baselines.hopcroft_tarjan(g)
        assert ht.num_bccs == lab.num_bccs, name
        names.append(name); ns.append(n); ms.append(g.m)
        ks.append(res.forest_edges.pairs.shape[0]); es.append(el.size)
        cols["offsets"].append(g.offsets.astype(np.int64))
        cols["edges"].append(g.edges.astype(np.uint32))
        cols["cc_label"].append(res.labels.astype(np.int32))
        cols["forest"].append(res.forest_edges.pairs.astype(np.int32).reshape(-1, 2))
        for k in ("parent", "first", "last"):
            cols[k].append(getattr(f, k).astype(np.int32))
        for k in ("w1", "w2", "low", "high"):
            cols[k].append(getattr(tags, k).astype(np.int32))
        cols["fence"].append((skel[:, 1] & 1).astype(np.uint8) if n else np.empty(0, np.uint8))
        cols["label"].append(lab.label.astype(np.int32))
        cols["head"].append(lab.head.astype(np.int32))
        cols["is_ap"].append(ap)
        cols["edge_label"].append(el)
        nbccs.append(lab.num_bccs); ncomps.append(lab.num_components)
        ht_nbccs.append(ht.num_bccs)
    out = {k: np.concatenate(v) if v else np.empty(0) for k, v in cols.items()}
    out["forest"] = np.concatenate(cols["forest"]).reshape(-1, 2)
    out.update(names=np.array(names), n=np.array(ns, np.int64), m=np.array(ms, np.int64),
               k=np.array(ks, np.int64), E=np.array(es, np.int64),
               num_bccs=np.array(nbccs, np.int64), num_components=np.array(ncomps, np.int64),
               ht_num_bccs=np.array(ht_nbccs, np.int64))
    np.savez_compressed(HERE / "corpus.npz", **out)
    print(f"corpus: {len(names)} graphs, {int(np.sum(ns))} vertices, {int(np.sum(ms))} slots")


def classify(fb):
    """classify.npz: the reference's edge classes on the corpus, for the
    reference's own rooted forest and tags stored in corpus.npz -- per upper
    arc (u < v) in CSR order, EdgeClass values (bcc.py:45-51): PLAIN_TREE 0,
    FENCE_TREE 1, BACK 2, CROSS 3.  Each class comes from bcc.classify_edge
    (bcc.py:54-70) and is asserted equal to the first-principles
    tests/oracles.py classify_edges_oracle (oracles.py:207-235)."""
    import importlib.util

    import oracles  # the reference's (its tests dir is on sys.path)
    from fastbcc import bcc, euler_tour, graphs as rg, tagging

    spec = importlib.util.spec_from_file_location("repo_conftest", REPO / "tests" / "conftest.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    c = mod.Corpus(HERE / "corpus.npz")
    code = {"plain": 0, "fence": 1, "back": 2, "cross": 3}
    cls_all, counts = [], []
    for i, name, g in c.items():
        n = g.n
        gr = rg.Graph(g.offsets, g.edges)
        parent, first, last = (c.get(i, k) for k in ("parent", "first", "last"))
        roots = np.flatnonzero(parent == -1)
        forest = euler_tour.RootedForest(parent, first, last, roots)
        tags = tagging.VertexTags(*(c.get(i, k) for k in ("w1", "w2", "low", "high")))
        want = oracles.classify_edges_oracle(gr, parent) if n else {}
        out = []
        for u in range(n):
            for v in g.edges[g.offsets[u]:g.offsets[u + 1]]:
                v = int(v)
                if u > v:
                    continue
                k = int(bcc.classify_edge(forest, tags, u, v))
                assert k == code[want[(u, v)]], (name, u, v)
                out.append(k)
        cls_all.append(np.array(out, np.int8))
        counts.append(len(out))
    np.savez_compressed(HERE / "classify.npz", cls=np.concatenate(cls_all), E=np.array(counts, np.int64))
    print(f"classify: {len(counts)} graphs, {int(np.sum(counts))} edges")
    # extract.npz: the reference's extract_bccs (bcc.py:199-219) on the
    # reference's labeling of every corpus graph
    verts, blens, nblocks = [], [], []
    for i, name, g in c.items():
        lab = bcc.BccLabeling(c.get(i, "label"), c.get(i, "head"), c.get(i, "num_bccs"),
                              c.get(i, "num_components"), bcc.StepTimings())
        blocks = bcc.extract_bccs(lab)
        nblocks.append(len(blocks))
        for b in blocks:
            verts.append(np.asarray(b, np.int32))
            blens.append(len(b))
    np.savez_compressed(HERE / "extract.npz", verts=np.concatenate(verts) if verts else np.empty(0, np.int32),
                        blen=np.array(blens, np.int64), nblocks=np.array(nblocks, np.int64))
    print(f"extract: {int(np.sum(nblocks))} blocks")


def listrank(fb):
    from fastbcc.euler_tour import list_ranking

    rng = np.random.Generator(np.random.PCG64(2024))
    nxts, heads, ranks, Ls, Hs = [], [], [], [], []
    for trial in range(40):
        L = int(rng.integers(1, 3000))
        perm = rng.permutation(L)
        nl = int(rng.integers(1, 9))
        cuts = np.sort(rng.choice(np.arange(1, L), size=min(nl - 1, L - 1), replace=False)) if L > 1 else np.array([], int)
        nxt = np.full(L, -1, np.int32)
        hs = []
        for piece in np.split(perm, cuts):
            hs.append(piece[0])
            nxt[piece[:-1]] = piece[1:]
        hs = np.array(hs + [-1], np.int32)  # a trailing ignored head
        r = list_ranking(nxt, hs)
        nxts.append(nxt); heads.append(hs); ranks.append(r.astype(np.int32))
        Ls.append(L); Hs.append(hs.size)
    # error cases (test_euler_tour.py:143-162): each must raise ValueError
    bad = [([1, 2, 0], [0]), ([-1, -1], [0]), ([2, 2, -1], [0, 1]), ([1, 2, -1], [0, 1])]
    for nx, hd in bad:
        try:
            list_ranking(np.array(nx, np.int32), np.array(hd, np.int32))
            raise AssertionError("reference accepted a bad list")
        except ValueError:
            pass
    np.savez_compressed(HERE / "listrank.npz", nxt=np.concatenate(nxts), heads=np.concatenate(heads),
                        ranks=np.concatenate(ranks), L=np.array(Ls, np.int64), H=np.array(Hs, np.int64),
                        bad_nxt=np.array([np.array(b[0], np.int32) for b in bad], dtype=object),
                        bad_heads=np.array([np.array(b[1], np.int32) for b in bad], dtype=object))
    print(f"listrank: {len(Ls)} cases")


def configs(fb, names=("1", "2", "3")):
    sys.path.insert(0, str(REPO))
    import workloads
    from fastbcc import baselines, bcc, graphs as rg

    meta = {}
    for name in names:
        t0 = time.time()
        mine = workloads.make(name)
        g = rg.Graph(mine.offsets, mine.edges)
        lab = bcc.fast_bcc(g)
        ap = np.zeros(g.n, np.uint8)
        ap[bcc.articulation_points(lab)] = 1
        el = canonical_edge_labels(g, lab.label, lab.head)
        if name in ("1", "2", "3"):
            tv = baselines.tv_skeleton(g).edge_label
            assert np.array_equal(tv.astype(np.int64), el.astype(np.int64)), name
        meta[name] = dict(desc=workloads.CONFIGS[name][0], n=g.n, m=g.m, E=int(el.size),
                          csr_sha256=workloads.csr_digest(mine), num_bccs=int(lab.num_bccs),
                          num_components=int(lab.num_components), num_ap=int(ap.sum()),
                          label_sha256=sha(lab.label.astype(np.int32)),
                          head_sha256=sha(lab.head.astype(np.int32)),
                          is_ap_sha256=sha(ap), edge_label_sha256=sha(el.astype(np.int32)),
                          ref_seconds=float(lab.timings.total))
        if name == "1":
            np.savez_compressed(HERE / "config1.npz", label=lab.label.astype(np.int32),
                                head=lab.head.astype(np.int32), is_ap=ap, edge_label=el)
        print(f"config {name}: {meta[name]['num_bccs']} BCCs, {meta[name]['num_ap']} APs, "
              f"{meta[name]['num_components']} comps ({time.time() - t0:.1f}s)")
    path = HERE / "configs.json"
    old = json.loads(path.read_text()) if path.exists() else {}
    old.update(meta)
    path.write_text(json.dumps(old, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-configs", action="store_true")
    ap.add_argument("--configs", default="1,2,3")
    ap.add_argument("--only-configs", action="store_true")
    ap.add_argument("--only-classify", action="store_true")
    a = ap.parse_args()
    fb = import_reference()
    if a.only_classify:
        classify(fb)
        sys.exit(0)
    if not a.only_configs:
        corpus(fb)
        listrank(fb)
    if not a.skip_configs:
        configs(fb, a.configs.split(","))
