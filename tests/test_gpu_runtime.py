"""Device all-reduce of the rank runtime (Comm.all_reduce_sum, runtime.py
of the reference): ascending-rank sums, bit-identical on every member,
subgroups independent, ring-convention ledger charges."""

import numpy as np
import pytest
import torch

import paper_2504_04673_b200 as P

pytestmark = pytest.mark.gpu


def test_allreduce_group_of_one_and_pair():
    res = P.run_program(1, 1, lambda comm: comm.all_reduce_sum(np.arange(3.0)))
    assert np.array_equal(res.results[0], np.arange(3.0))
    res = P.run_program(2, 1, lambda comm: comm.all_reduce_sum(np.full(4, comm.rank + 1.0)))
    for out in res.results:
        assert np.array_equal(out, np.full(4, 3.0))


def test_allreduce_matches_sequential_sum_bitwise():
    p = 5
    data = [np.random.default_rng(r).standard_normal(257).astype(np.float32) for r in range(p)]

    def prog(comm):
        return comm.all_reduce_sum(torch.from_numpy(data[comm.rank]).cuda())

    res = P.run_program(p, 1, prog)
    ref = torch.from_numpy(data[0]).cuda()
    for r in range(1, p):
        ref = ref + torch.from_numpy(data[r]).cuda()          # ascending rank order
    for out in res.results:
        assert torch.equal(out, ref)


def test_subgroup_allreduce_independent():
    def prog(comm):
        grp = comm.grid.col_group(comm.coords[1])
        return comm.all_reduce_sum(np.full(3, float(comm.rank)), group=grp)

    res = P.run_program(4, 2, prog)
    assert np.array_equal(res.results[0], np.full(3, 2.0))   # ranks 0 + 2
    assert np.array_equal(res.results[1], np.full(3, 4.0))   # ranks 1 + 3


def test_allreduce_rejects_shape_mismatch():
    with pytest.raises(ValueError):
        P.run_program(2, 1, lambda comm: comm.all_reduce_sum(np.zeros(2 + comm.rank)))
