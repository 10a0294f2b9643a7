"""The radius-query oracle (oracle.neighbor_csr) pinned to the reference's own
tables (tests/golden/nbr_*.npz, made by tests/golden/make_golden_neighbors.py),
and the uid-space table hash (spatial.neighbor_table_hash) pinned to the
reference's digest."""

import glob
import os

import numpy as np
import pytest

from oracle import oracle
from paper_2105_00039_b200 import spatial

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "nbr_*.npz")))


class _Pool:
    def __init__(self, g):
        self.uid = g["uid"]


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[4:-4] for p in GOLDEN])
def test_oracle_matches_reference_table(path):
    g = np.load(path)
    indptr, indices = oracle.neighbor_csr(g["px"], g["py"], g["pz"], g["uid"], float(g["radius"]))
    assert np.array_equal(indptr, g["indptr"])
    assert np.array_equal(indices, g["indices"])
    assert np.array_equal(np.diff(indptr), g["counts"])


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[4:-4] for p in GOLDEN])
def test_table_hash_matches_reference(path):
    g = np.load(path)
    assert spatial.neighbor_table_hash(_Pool(g), g["indptr"], g["indices"]) == str(g["table_hash"])


def test_golden_cover_edge_cases():
    names = {os.path.basename(p) for p in GOLDEN}
    assert {"nbr_degenerate_f64.npz", "nbr_single_f64.npz", "nbr_rand_f32.npz"} <= names
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "nbr_degenerate_f64.npz"))
    # coincident pair and pairs at exactly d == radius are neighbours (closed ball)
    assert g["counts"][0] >= 2 and g["indptr"][-1] == g["counts"].sum()
