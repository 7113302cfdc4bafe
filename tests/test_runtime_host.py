"""The rank runtime's host semantics (runtime.py of the reference): process
grid, buffered point-to-point with per-tag FIFO order, personalised
exchange, broadcast, ledger conventions (8 bytes per element, index vs data
traffic, pair maxima, marks), error reporting.  Host payloads only."""

import numpy as np
import pytest

import paper_2504_04673_b200 as P


def test_grid_layout_and_groups():
    g = P.ProcessGrid(8, 2)
    assert g.n_rows == 4 and g.rank_of(3, 1) == 7 and g.coords(5) == (2, 1)
    assert g.row_group(1) == (2, 3) and g.col_group(1) == (1, 3, 5, 7)
    assert P.ProcessGrid(8, 2).stage_count() == 2


@pytest.mark.parametrize("p,c", [(0, 1), (4, 0), (6, 4)])
def test_grid_rejects_bad_shapes(p, c):
    with pytest.raises(ValueError):
        P.ProcessGrid(p, c)


def test_single_rank_program_and_self_send_free():
    def prog(comm):
        comm.isend(0, np.arange(4.0))
        return comm.recv(0).sum()

    res = P.run_program(1, 1, prog)
    assert res.results == [6.0]
    assert res.ledger.total_bytes_sent() == 0          # a self-send is free


def test_ring_bytes_and_fifo_per_tag():
    def prog(comm):
        r, p = comm.rank, comm.p
        for k in range(3):
            comm.isend((r + 1) % p, np.full(2, 10.0 * k + r), tag="a")
        comm.isend((r + 1) % p, np.full(5, -1.0), tag="b")
        got_b = comm.recv((r - 1) % p, tag="b")
        got_a = [comm.recv((r - 1) % p, tag="a")[0] for _ in range(3)]
        return got_a, float(got_b.sum())

    res = P.run_program(3, 1, prog)
    for r, (a, b) in enumerate(res.results):
        src = (r - 1) % 3
        assert a == [10.0 * k + src for k in range(3)] and b == -5.0
    c = res.ledger.counters["p2p"]
    assert c["data_bytes_sent"].tolist() == [8.0 * (3 * 2 + 5)] * 3
    assert c["msgs_sent"].tolist() == [4] * 3


def test_zero_length_payload_delivered_free():
    def prog(comm):
        if comm.rank == 0:
            comm.isend(1, np.zeros(0))
            return None
        return comm.recv(0).size

    res = P.run_program(2, 1, prog)
    assert res.results[1] == 0
    assert res.ledger.counters["p2p"]["data_bytes_sent"].sum() == 0


def test_alltoallv_matches_sequential_exchange():
    p = 4

    def prog(comm):
        bufs = [np.full(d + 1, 100.0 * comm.rank + d) for d in range(p)]
        return comm.all_to_allv(bufs)

    res = P.run_program(p, 1, prog)
    for r in range(p):
        for s in range(p):
            assert np.array_equal(res.results[r][s], np.full(r + 1, 100.0 * s + r))


def test_broadcast_bit_identical_and_linear_at_root():
    p = 4
    data = np.random.default_rng(0).standard_normal(6)

    def prog(comm):
        return comm.broadcast(2, data if comm.rank == 2 else None)

    res = P.run_program(p, 1, prog)
    for out in res.results:
        assert np.array_equal(out, data)
    sent = res.ledger.counters["broadcast"]["bytes_sent"]
    assert sent[2] == 8 * 6 * (p - 1) and sent.sum() == sent[2]
    with pytest.raises(ValueError):
        P.run_program(2, 1, lambda comm: comm.broadcast(5, np.zeros(1)))


def test_deadlock_and_leftover_messages_and_exceptions():
    with pytest.raises(P.DeadlockError):
        P.run_program(2, 1, lambda comm: comm.recv(1 - comm.rank))

    def leftover(comm):
        if comm.rank == 1:
            comm.isend(0, np.ones(3))

    with pytest.raises(P.SimulationError):
        P.run_program(2, 1, leftover)

    def boom(comm):
        if comm.rank == 1:
            raise RuntimeError("rank 1 failed")
        comm.recv(1)

    with pytest.raises(RuntimeError, match="rank 1 failed"):
        P.run_program(2, 1, boom)


def test_payload_types():
    with pytest.raises(TypeError):
        P.run_program(2, 1, lambda comm: comm.isend(1 - comm.rank, np.array(["x"])))


def test_index_traffic_and_pair_max_and_marks():
    def prog(comm):
        if comm.rank == 0:
            comm.isend(1, np.arange(3, dtype=np.int64))
            comm.isend(1, np.zeros(7))
            comm.isend(1, np.zeros(2))
        else:
            for _ in range(3):
                comm.recv(0)
        comm.ledger_mark("after")

    res = P.run_program(2, 1, prog)
    c = res.ledger.counters["p2p"]
    assert c["index_bytes_sent"][0] == 24 and c["data_bytes_sent"][0] == 72
    assert res.ledger.pair_max_data_bytes[(0, 1)] == 56
    assert res.ledger.marks["after"]["p2p"]["bytes_sent"] == 96


def test_runs_deterministic():
    def prog(comm):
        comm.isend((comm.rank + 1) % comm.p, np.full(3, float(comm.rank)))
        return comm.recv((comm.rank - 1) % comm.p).tolist()

    a, b = P.run_program(4, 1, prog), P.run_program(4, 1, prog)
    assert a.results == b.results and a.ledger.to_dict() == b.ledger.to_dict()


@pytest.mark.parametrize("kw", [dict(layers=1), dict(hidden=0), dict(lr=-0.1), dict(epochs=-1),
                                dict(activation="tanh"), dict(order="sideways")])
def test_train_config_validation(kw):
    with pytest.raises(ValueError):
        P.TrainConfig(**kw)


def test_train_config_layer_dims():
    cfg = P.TrainConfig(layers=4, hidden=16)
    assert cfg.layer_dims(100, 47) == [100, 16, 16, 47]       # 3 weight matrices
