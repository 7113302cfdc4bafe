"""Reference-API behaviour of the CUDA path: edge cases (empty parts,
empty rows, no nonzeros), error messages, user rank programs calling
spmm_kernel / all_reduce_sum, tensor in -> tensor out."""

import numpy as np
import pytest
import torch

import distgcn_oracle as O
import paper_2504_04673_b200 as P

pytestmark = pytest.mark.gpu


def _ref(d, h):
    return O.serial_reference(O.csr_from_dense(d), h)


def test_empty_part_and_empty_rows():
    rng = np.random.default_rng(3)
    n = 30
    d = rng.normal(size=(n, n)) * (rng.random((n, n)) < 0.15)
    d[5, :] = 0.0
    d[:, 7] = 0.0
    h = rng.normal(size=(n, 5)).astype(np.float32).astype(np.float64)
    d = d.astype(np.float32).astype(np.float64)
    asg = rng.integers(0, 3, size=n)             # part 3 of 4 stays empty
    part = P.Partition.from_assignment(asg, 4)
    for variant, p, c in [("1d-sparse", 4, 1), ("1d-oblivious", 4, 1), ("15d-sparse", 8, 2)]:
        run = P.run_spmm(P.csr_from_dense(d), h, p, c, variant, partition=part)
        np.testing.assert_allclose(run.z, _ref(d, h), rtol=1e-5, atol=1e-6)


def test_no_nonzeros():
    d = np.zeros((12, 12))
    h = np.ones((12, 3))
    run = P.run_spmm(P.csr_from_dense(d), h, 4, 1, "1d-sparse")
    assert not run.z.any()
    assert run.ledger.total_bytes_sent() == 0.0


def test_errors_match_reference_messages():
    a = P.csr_from_dense(np.eye(4))
    with pytest.raises(ValueError, match="dimension mismatch"):
        P.local_spmm(a, np.ones((3, 2)))
    with pytest.raises(ValueError, match="dimension mismatch"):
        P.gemm(np.ones((2, 3)), np.ones((2, 3)))
    with pytest.raises(ValueError, match="parts"):
        P.run_spmm(P.csr_from_dense(np.eye(16)), np.ones((16, 2)), 4, 1, "1d-sparse",
                   partition=P.block_partition(16, 3))
    with pytest.raises(ValueError, match="square"):
        P.run_spmm(P.csr_from_dense(np.ones((3, 4))), np.ones((3, 2)), 1, 1, "1d-sparse")


def test_user_program_calls_spmm_kernel_and_allreduce():
    """The reference's usage pattern: rank programs under run_program."""
    rng = np.random.default_rng(9)
    n = 24
    d = rng.normal(size=(n, n)) * (rng.random((n, n)) < 0.2)
    d = d.astype(np.float32).astype(np.float64)
    h = rng.normal(size=(n, 4)).astype(np.float32).astype(np.float64)
    a = P.csr_from_dense(d)
    grid = P.ProcessGrid(4, 1)
    part = P.block_partition(n, 4)
    dm = P.build_dist_matrices(a, part.boundaries, grid)

    def program(comm):
        r0, r1 = dm.boundaries[comm.rank]
        P.exchange_index_lists(comm, dm.fwd, "1d-sparse")
        z = P.spmm_kernel(comm, dm.fwd, h[r0:r1], "1d-sparse")
        s = comm.all_reduce_sum(np.array([z.sum()]))
        return z, s

    run = P.run_program(4, 1, program)
    z = np.vstack([run.results[r][0] for r in range(4)])
    np.testing.assert_allclose(z, _ref(d, h), rtol=1e-5, atol=1e-6)
    sums = [run.results[r][1] for r in range(4)]
    assert all(np.array_equal(sums[0], s) for s in sums)
    assert run.ledger.counters["allreduce"]["calls"].tolist() == [1, 1, 1, 1]


def test_tensor_in_tensor_out():
    rng = np.random.default_rng(1)
    n = 40
    d = rng.normal(size=(n, n)) * (rng.random((n, n)) < 0.1)
    d = d.astype(np.float32).astype(np.float64)
    h = torch.randn(n, 6, device="cuda")
    run = P.run_spmm(P.csr_from_dense(d), h, 2, 1, "1d-sparse")
    assert isinstance(run.z, torch.Tensor) and run.z.is_cuda
    np.testing.assert_allclose(run.z.double().cpu().numpy(), _ref(d, h.double().cpu().numpy()),
                               rtol=1e-5, atol=1e-6)


def test_f_not_multiple_of_four_and_wide():
    rng = np.random.default_rng(2)
    n = 50
    d = (rng.normal(size=(n, n)) * (rng.random((n, n)) < 0.2)).astype(np.float32).astype(float)
    for f in (1, 5, 67, 130, 602):
        h = rng.normal(size=(n, f)).astype(np.float32).astype(np.float64)
        z = P.local_spmm(P.csr_from_dense(d), h)
        ref = O.local_spmm(O.csr_from_dense(d), h)
        mag = O.local_spmm(O.csr_from_dense(np.abs(d)), np.abs(h))
        assert np.all(np.abs(z - ref) <= 1e-5 * mag + 1e-30), f


def test_run_graph_equals_eager_run():
    """The CUDA-graph-captured epoch (GcnRun.run_graph) replays exactly the
    eager epoch: losses, weights and ledger marks bit-identical."""
    from paper_2504_04673_b200 import graphgen
    from paper_2504_04673_b200.gcn import GcnRun
    a = P.gcn_normalize(graphgen.rmat(10, 8, 2))
    a.values = a.values.astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((a.n_rows, 24)).astype(np.float32)
    y = rng.integers(0, 5, a.n_rows)
    cfg = P.TrainConfig(layers=3, hidden=16, lr=0.1, epochs=4, seed=1)
    gr = GcnRun(a, x, y, np.ones(a.n_rows, bool), cfg)
    ref = gr.result(gr.run())
    for _ in range(2):                               # capture once, replay twice
        got = gr.result(gr.run_graph())
        assert np.array_equal(got.losses, ref.losses)
        for w1, w2 in zip(got.weights, ref.weights):
            assert np.array_equal(w1, w2)
        assert got.history == ref.history
    gr.close()


@pytest.mark.parametrize("p,c,variant", [(4, 1, "1d-sparse"), (4, 2, "15d-sparse"),
                                         (3, 1, "1d-oblivious")])
def test_run_lockstep_equals_threaded_run(p, c, variant):
    """One host thread driving every hosted rank in lock step gives the
    thread-per-rank runtime's results bit for bit, ledger included."""
    from paper_2504_04673_b200 import graphgen
    from paper_2504_04673_b200.gcn import GcnRun
    a = P.gcn_normalize(graphgen.rmat(10, 8, 4))
    a.values = a.values.astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((a.n_rows, 20)).astype(np.float32)
    y = rng.integers(0, 7, a.n_rows)
    cfg = P.TrainConfig(layers=4, hidden=16, lr=0.1, epochs=3, seed=2, variant=variant)
    gr = GcnRun(a, x, y, np.ones(a.n_rows, bool), cfg, p=p, c=c)
    ref = gr.result(gr.run())
    got = gr.result(gr.run_lockstep())
    gr.close()
    assert np.array_equal(got.losses, ref.losses)
    for w1, w2 in zip(got.weights_per_rank, ref.weights_per_rank):
        for a1, a2 in zip(w1, w2):
            assert np.array_equal(a1, a2)
    assert got.history == ref.history
    for prim in ref.ledger.counters:
        for name, v in ref.ledger.counters[prim].items():
            assert np.array_equal(got.ledger.counters[prim][name], v), (prim, name)
    assert got.ledger.pair_max_bytes == ref.ledger.pair_max_bytes


def test_run_graph_multi_rank_equals_eager():
    """Four ranks in one process: the captured lock-step epoch replays the
    threaded runtime's results bit for bit, ledger included."""
    from paper_2504_04673_b200 import graphgen
    from paper_2504_04673_b200.gcn import GcnRun
    a = P.gcn_normalize(graphgen.rmat(10, 8, 9))
    a.values = a.values.astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(5)
    x = rng.standard_normal((a.n_rows, 16)).astype(np.float32)
    y = rng.integers(0, 4, a.n_rows)
    cfg = P.TrainConfig(layers=3, hidden=16, lr=0.1, epochs=3, seed=4, variant="1d-sparse")
    gr = GcnRun(a, x, y, np.ones(a.n_rows, bool), cfg, p=4)
    ref = gr.result(gr.run())
    for _ in range(2):
        got = gr.result(gr.run_graph())
        assert np.array_equal(got.losses, ref.losses)
        for w1, w2 in zip(got.weights_per_rank, ref.weights_per_rank):
            for a1, a2 in zip(w1, w2):
                assert np.array_equal(a1, a2)
        assert got.history == ref.history
        for prim in ref.ledger.counters:
            for name, v in ref.ledger.counters[prim].items():
                assert np.array_equal(got.ledger.counters[prim][name], v), (prim, name)
    gr.close()
