"""Shared fixtures.  ``-m gpu`` tests need a B200; everything else runs on CPU.

Golden fixtures under tests/golden/ were produced by running the reference
package itself (tests/golden/make_golden.py); they are the parity anchor.
"""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


class Corpus:
    """The reference test corpus with the reference's outputs, per graph."""

    def __init__(self, path):
        z = np.load(path, allow_pickle=False)
        self.z = {k: z[k] for k in z.files}
        self.names = [str(s) for s in self.z["names"]]
        n, m, k, E = (self.z[x] for x in ("n", "m", "k", "E"))
        self._on = np.concatenate([[0], np.cumsum(n + 1)])
        self._vn = np.concatenate([[0], np.cumsum(n)])
        self._em = np.concatenate([[0], np.cumsum(m)])
        self._fk = np.concatenate([[0], np.cumsum(k)])
        self._ee = np.concatenate([[0], np.cumsum(E)])

    def __len__(self):
        return len(self.names)

    def graph(self, i):
        from paper_2301_01356_b200.graphs import Graph

        z = self.z
        return Graph(z["offsets"][self._on[i]:self._on[i + 1]], z["edges"][self._em[i]:self._em[i + 1]])

    def get(self, i, key):
        z = self.z
        if key in ("forest",):
            return z[key][self._fk[i]:self._fk[i + 1]]
        if key == "edge_label":
            return z[key][self._ee[i]:self._ee[i + 1]]
        if key in ("num_bccs", "num_components", "ht_num_bccs", "n", "m", "k", "E"):
            return int(z[key][i])
        return z[key][self._vn[i]:self._vn[i + 1]]

    def items(self):
        for i, name in enumerate(self.names):
            yield i, name, self.graph(i)


@pytest.fixture(scope="session")
def corpus():
    return Corpus(GOLDEN / "corpus.npz")


@pytest.fixture(scope="session")
def config_meta():
    return json.loads((GOLDEN / "configs.json").read_text())


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle

    oracle.build()
    return oracle


def relaxed_w2(offsets, edges, parent, first):
    """w2 as the fused pipeline computes it (tags.cu, WGatherVisitor<false>):
    max(first[v], first[w]) over neighbours w except the tree parent -- tree
    children are kept.  The exact w2 of tagging.py:101-119 excludes them too;
    both give the same w1, low and high (checked in the rung-3 tests)."""
    n = len(offsets) - 1
    deg = np.diff(offsets).astype(np.int64)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    dst = np.asarray(edges, dtype=np.int64)
    keep = dst != np.asarray(parent, dtype=np.int64)[src]
    w2 = np.asarray(first, dtype=np.int64).copy()
    np.maximum.at(w2, src[keep], np.asarray(first, dtype=np.int64)[dst[keep]])
    return w2.astype(np.int32)
