"""The host CSR generator (tools/hostgen.c) reproduces workloads.rmat() and
graphs.symmetrize() bit for bit -- the bench builds config 5 with it."""

import numpy as np
import pytest

import workloads
from paper_2301_01356_b200.graphs import symmetrize


@pytest.mark.parametrize("scale,ef,chunk,seed", [(10, 16, 1 << 24, 0), (12, 8, 5000, 3), (14, 16, 1 << 16, 0)])
def test_rmat_fast_matches_numpy(scale, ef, chunk, seed):
    a = workloads.rmat(scale, ef, seed=seed, chunk=chunk)
    b = workloads.rmat_fast(scale, ef, seed=seed, chunk=chunk)
    assert workloads.csr_digest(a) == workloads.csr_digest(b)


def test_symmetrize_host_matches_symmetrize():
    rng = np.random.default_rng(7)
    n = 3000
    pairs = rng.integers(0, n, size=(40000, 2))
    pairs[:50, 1] = pairs[:50, 0]  # self-loops
    pairs = np.concatenate([pairs, pairs[:1000]])  # duplicates
    a = symmetrize(pairs, n)
    b = workloads.symmetrize_host(pairs[:, 0], pairs[:, 1], n)
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.edges, b.edges)
    with pytest.raises(ValueError):
        workloads.symmetrize_host(np.array([0, n]), np.array([1, 2]), n)
    e = workloads.symmetrize_host(np.zeros(0), np.zeros(0), 5)
    assert e.n == 5 and e.m == 0
