"""Locality schedules (locality.py) on CPU: label propagation recovers
planted communities, lpa_partition is a valid balanced partition, the row
order is a permutation.  The GPU side (same results bit for bit with and
without the order) is in tests/test_gpu_locality.py."""

import numpy as np
import pytest
import torch

import paper_2504_04673_b200 as P
from paper_2504_04673_b200 import graphgen
from paper_2504_04673_b200.locality import (_edges, community_order, label_propagation,
                                            lpa_partition, rank_row_order)

CPU = torch.device("cpu")


@pytest.fixture(scope="module")
def planted():
    n = 40_000
    a, comm = graphgen.chung_lu_device(n, n * 20, alpha=0.55, max_weight=300, seed=3,
                                       communities=32, p_in=0.8, return_communities=True,
                                       device=CPU)
    return a, comm


def test_label_propagation_recovers_planted_communities(planted):
    a, comm = planted
    rows, cols = _edges(a.row_ptr, a.col_idx, a.n_rows, CPU)
    lab = label_propagation(rows, cols, a.n_rows).numpy()
    # every label is (almost) pure in one planted community, and the labels
    # keep the planted share of intra-community edges
    pure = sum(np.bincount(comm[lab == u]).max() for u in np.unique(lab))
    assert pure / a.n_rows > 0.99
    r, c = rows.numpy(), cols.numpy()
    assert (lab[r] == lab[c]).mean() >= 0.97 * (comm[r] == comm[c]).mean()
    # deterministic
    lab2 = label_propagation(rows, cols, a.n_rows).numpy()
    assert np.array_equal(lab, lab2)


def test_community_order_is_grouped_permutation():
    lab = torch.tensor([5, 2, 5, 7, 2, 2, 7, 5])
    o = community_order(lab)
    assert o.dtype == np.int32 and sorted(o.tolist()) == list(range(8))
    # groups in order of their first row, rows ascending inside a group
    assert o.tolist() == [0, 2, 7, 1, 4, 5, 3, 6]


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_lpa_partition_balanced_and_cuts_less_than_block(planted, k):
    a, _ = planted
    part = lpa_partition(a, k, device=CPU)
    part.validate()
    deg = np.diff(a.row_ptr) + 1
    share = np.bincount(part.assignment, weights=deg, minlength=k) / deg.sum()
    assert share.max() <= 1.0 / k * 1.1
    # every part is contiguous in the layout, as Partition requires
    for q, (s, e) in enumerate(part.boundaries):
        assert np.all(part.assignment[np.argsort(part.perm)[s:e]] == q)
    if k > 1:
        # edge cut: the planted graph's 20% random edges, not the block
        # partition's (k-1)/k of all edges
        rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_ptr))
        cut = (part.assignment[rows] != part.assignment[a.col_idx]).mean()
        assert cut < 0.3 * (k - 1) / k
        assert P.comm_metrics(a, part, 1).total_rows <= \
            P.comm_metrics(a, P.block_partition(a.n_rows, k), 1).total_rows


def test_rank_row_order(planted):
    a, _ = planted

    class RO:
        n_rows = n_local = a.n_rows
        row_ptr = a.row_ptr
        col_ext = a.col_idx.astype(np.int32)

    o = rank_row_order(RO, "lpa", CPU)
    assert o.dtype == np.int32 and np.array_equal(np.sort(o), np.arange(a.n_rows))
    assert rank_row_order(RO, None, CPU) is None
    with pytest.raises(ValueError):
        rank_row_order(RO, "metis", CPU)
