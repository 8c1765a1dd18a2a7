"""Pins of oracle/binning.py (block partition)."""

import fractions
import json
import math
import os

import numpy as np

from oracle import binning
from paper_2208_00049_b200 import workloads

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_spec_example():
    g = GOLDEN["binning"]
    key, P = binning.tile_keys(np.array([[g["k"]]]), (g["Ntilde"],), (g["Q"],))
    assert P == (4,)
    assert key[0] == g["tile"]


def test_key_equals_block_membership_formula():
    """With P Q = Ntilde (power of two), the integer form equals the block
    membership k in R_p <=> p = floor((k + 1/2) P)."""
    rng = np.random.default_rng(0)
    nodes = workloads.uniform_nodes(rng, 5000, 2)
    Ntilde, Q = (64, 128), (16, 32)
    key, P = binning.tile_keys(nodes, Ntilde, Q)
    p0 = np.floor((nodes[:, 0] + 0.5) * P[0]).astype(int)
    p1 = np.floor((nodes[:, 1] + 0.5) * P[1]).astype(int)
    np.testing.assert_array_equal(key, p0 * P[1] + p1)


def test_perm_is_stable_sort_and_offsets_are_counts():
    rng = np.random.default_rng(1)
    nodes = workloads.uniform_nodes(rng, 3000, 3)
    Ntilde, Q = (16, 20, 24), (4, 7, 24)
    perm, offsets, P = binning.bin_nodes(nodes, Ntilde, Q)
    key, _ = binning.tile_keys(nodes, Ntilde, Q)
    assert P == (4, 3, 1)
    assert sorted(perm.tolist()) == list(range(3000))
    ks = key[perm]
    assert np.all(np.diff(ks) >= 0)
    same = np.diff(ks) == 0
    assert np.all(np.diff(perm)[same] > 0)  # ties in original order
    for p in range(int(np.prod(P))):
        assert offsets[p + 1] - offsets[p] == np.sum(key == p)


def test_single_tile_is_identity():
    rng = np.random.default_rng(2)
    nodes = workloads.uniform_nodes(rng, 100, 1)
    perm, offsets, P = binning.bin_nodes(nodes, (64,), (64,))
    assert P == (1,)
    np.testing.assert_array_equal(perm, np.arange(100))
    assert offsets.tolist() == [0, 100]


def test_fp32_nodes_cell_is_exact():
    """For fp32 nodes t = Ntilde k is computed in fp64, which is exact
    (24 + 9 bits < 53), so a = floor(t) is the exact rational floor (R11)."""
    nodes = workloads.radial_nodes(dtype=np.float32)
    for nt in (320, 512):
        t = float(nt) * nodes.astype(np.float64)
        sample = np.random.default_rng(3).choice(nodes.size, 2000, replace=False)
        flat = nodes.reshape(-1)
        for s in sample:
            exact = math.floor(fractions.Fraction(nt) * fractions.Fraction(float(flat[s])))
            assert math.floor(t.reshape(-1)[s]) == exact
