"""Property tests of the host plan builder against the oracle (CPU):
NnzCols lists and ledger volumes on random instances, every variant,
including empty parts and empty rows (hypothesis, like test_sparse.py:160)."""

import numpy as np
from hypothesis import given, settings, strategies as st

import distgcn_oracle as O
import paper_2504_04673_b200 as P
from paper_2504_04673_b200.plan import build_variant_plan, index_setup_charges
from paper_2504_04673_b200.runtime import CommLedger, ProcessGrid

GRIDS = [("1d-sparse", 3, 1), ("1d-oblivious", 4, 1), ("15d-sparse", 4, 2),
         ("15d-oblivious", 8, 2), ("15d-sparse", 8, 2), ("15d-sparse", 4, 1)]


@settings(max_examples=40, deadline=None)
@given(seed=st.integers(0, 10_000), n=st.integers(5, 60), dens=st.floats(0.0, 0.3),
       g=st.integers(0, len(GRIDS) - 1), empty_part=st.booleans())
def test_plan_matches_oracle(seed, n, dens, g, empty_part):
    variant, p, c = GRIDS[g]
    nb = p // c
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(n, n)) * (rng.random((n, n)) < dens)
    a = P.csr_from_dense(d)
    asg = rng.integers(0, nb, size=n)
    if empty_part:
        asg[asg == nb - 1] = 0          # part nb-1 has no vertices
    part = P.Partition.from_assignment(asg, nb)
    a2, _ = P.apply_partition(a, None, part)
    grid = ProcessGrid(p, c)
    dm = P.build_dist_matrices(a2, part.boundaries, grid)
    oa = O.csr_from_dense(d)
    oa2, _, _ = O.apply_partition(oa, None, part.perm)
    fwd, _ = O.build_dist_matrices(oa2, part.boundaries)
    for key, cols in fwd["nnz_cols"].items():
        assert np.array_equal(dm.fwd.nnz_cols[key], cols)
    vp = build_variant_plan(dm.fwd, grid, variant)
    led = CommLedger(p)
    index_setup_charges(led, dm.fwd, grid, variant)
    vp.charge(led, 3)
    ol = O.Ledger(p)
    O.exchange_index_lists(ol, fwd, p, c, variant)
    hb = [np.zeros((e - s, 3)) for s, e in part.boundaries]
    O.spmm_all_ranks(ol, fwd, hb, p, c, variant)
    for prim in O.PRIMITIVES:
        for name in ("bytes_sent", "bytes_received", "msgs_sent", "msgs_received", "calls",
                     "data_bytes_sent", "index_bytes_sent"):
            assert np.array_equal(led.counters[prim][name], ol.counters[prim][name]), (prim, name)
    assert led.pair_max_data_bytes == ol.pair_max_data_bytes
