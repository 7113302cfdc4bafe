"""Host-side plan builder and runtime vs the reference's golden vectors
(no GPU): NnzCols lists bit-exact, ledger charges exact, grid contract."""

import numpy as np
import pytest

import paper_2504_04673_b200 as P
from paper_2504_04673_b200.plan import build_variant_plan, index_setup_charges
from paper_2504_04673_b200.runtime import CommLedger, ProcessGrid


def _part(g, key, n, k):
    asg = g[key + "__assign"] if k > 1 else np.zeros(n, np.int64)
    sizes = np.bincount(asg, minlength=k)
    bounds, pos = [], 0
    for s in sizes:
        bounds.append((pos, pos + int(s)))
        pos += int(s)
    return P.Partition(n, k, asg, g[key + "__perm"], bounds)


def _plan_ledger(g, key):
    a = g.csr(key + "__a", P.CsrMatrix)
    p, c, vi = (int(x) for x in g[key + "__cfg"])
    variant = P.VARIANTS[vi]
    part = _part(g, key, a.n_rows, p // c)
    a2, _ = P.apply_partition(a, None, part)
    grid = ProcessGrid(p, c)
    dm = P.build_dist_matrices(a2, part.boundaries, grid)
    vp = build_variant_plan(dm.fwd, grid, variant)
    led = CommLedger(p)
    index_setup_charges(led, dm.fwd, grid, variant)
    vp.charge(led, g[key + "__h"].shape[1])
    return a, p, c, variant, dm, vp, led


def test_nnz_cols_bit_exact(spmm_golden):
    g = spmm_golden
    for key in g.cases():
        _, p, c, _, dm, _, _ = _plan_ledger(g, key)
        nb = p // c
        cols = [dm.fwd.nnz_cols[(i, j)] for i in range(nb) for j in range(nb)]
        assert np.array_equal([x.size for x in cols], g[key + "__nnzc_len"]), key
        assert np.array_equal(np.concatenate(cols), g[key + "__nnzc"]), key


def test_ledger_exact(spmm_golden):
    g = spmm_golden
    for key in g.cases():
        _, p, c, variant, _, _, led = _plan_ledger(g, key)
        for (prim, name), ref in g.ledger_fields(key).items():
            assert np.array_equal(led.counters[prim][name], ref), (key, variant, prim, name)
        pm = np.array([[s, d, b] for (s, d), b in sorted(led.pair_max_data_bytes.items())],
                      dtype=np.float64).reshape(-1, 3)
        assert np.array_equal(pm, g[key + "__pairmax"]), key
        assert led.conservation_ok()


def test_rank_operands_reassemble_the_matrix(spmm_golden):
    """Every rank's remapped CSR, mapped back through its halo layout, is
    exactly its block row of A^T restricted to its stage band."""
    g = spmm_golden
    for key in g.cases():
        a, p, c, variant, dm, vp, _ = _plan_ledger(g, key)
        at = dm.fwd.mat.to_dense()
        grid = ProcessGrid(p, c)
        starts = dm.fwd.starts
        for ro in vp.ranks:
            r0, r1 = dm.boundaries[ro.i]
            # inverse of the ext map
            ext2glob = np.full(ro.n_local + ro.halo_rows, -1, dtype=np.int64)
            ext2glob[:ro.n_local] = np.arange(r0, r1)
            for q, off in ro.halo_off.items():
                rows = (dm.fwd.nnz_cols[(ro.i, q)] if variant.endswith("sparse")
                        else np.arange(dm.fwd.widths[q]))
                ext2glob[ro.n_local + off: ro.n_local + off + rows.size] = starts[q] + rows
            dense = np.zeros((ro.n_rows, at.shape[1]))
            rr = np.repeat(np.arange(ro.n_rows), np.diff(ro.row_ptr))
            gc = ext2glob[ro.col_ext]
            assert (gc >= 0).all()
            dense[rr, gc] = ro.val
            want = at[r0:r1].astype(np.float32)
            if variant.startswith("15d"):
                s = grid.stage_count()
                band = np.zeros(at.shape[1], bool)
                for q in range(ro.j * s, (ro.j + 1) * s):
                    band[starts[q]:starts[q + 1]] = True
                want = np.where(band[None, :], want, 0)
            assert np.array_equal(dense, want), (key, ro.rank)
        # every segment lands inside its receiver's halo
        for sgm in vp.segments:
            dst = vp.ranks[sgm.dst]
            assert sgm.dst_row0 + sgm.count <= dst.halo_rows


def test_1d_aware_volume_equals_comm_metrics(spmm_golden):
    g = spmm_golden
    for key in g.cases():
        if key + "__send_rows" not in g:
            continue
        a, p, c, variant, dm, vp, led = _plan_ledger(g, key)
        part = _part(g, key, a.n_rows, p)
        m = P.comm_metrics(a, part)
        assert np.array_equal(m.per_part_send_rows, g[key + "__send_rows"])
        f = g[key + "__h"].shape[1]
        assert vp.elements(f) == m.total_rows * f


def test_rmat14_volumes(rmat_volumes):
    """R-MAT-14 (config 1 graph) aware/oblivious volumes, 1D and 1.5D
    (c=2 and c=4 on 16 virtual ranks), equal to the reference's ledger."""
    g = rmat_volumes
    n = 16384
    from paper_2504_04673_b200.graphgen import rmat
    a = P.gcn_normalize(rmat(14, 16, 0))
    assert a.nnz == int(g["nnz"][0])
    assert np.array_equal(a.col_idx, g["ci"])
    for variant, p, c in [("1d-sparse", 4, 1), ("1d-oblivious", 4, 1), ("15d-sparse", 8, 2),
                          ("15d-sparse", 16, 4), ("15d-oblivious", 8, 2)]:
        grid = ProcessGrid(p, c)
        part = P.block_partition(n, grid.n_rows)
        dm = P.build_dist_matrices(a, part.boundaries, grid)
        vp = build_variant_plan(dm.fwd, grid, variant)
        led = CommLedger(p)
        index_setup_charges(led, dm.fwd, grid, variant)
        vp.charge(led, 16)
        for (prim, name), ref in g.ledger_fields(f"{variant}_{p}_{c}").items():
            assert np.array_equal(led.counters[prim][name], ref), (variant, prim, name)
    # 25,161 rows -> 3,220,608 B; oblivious 6,291,456 B (ratio 0.512)
    grid = ProcessGrid(4, 1)
    dm = P.build_dist_matrices(a, P.block_partition(n, 4).boundaries, grid)
    assert build_variant_plan(dm.fwd, grid, "1d-sparse").elements(16) * 8 == 3_220_608
    assert build_variant_plan(dm.fwd, grid, "1d-oblivious").elements(16) * 8 == 6_291_456


def test_variant_grid_validation_names_constraint():
    with pytest.raises(ValueError, match="c == 1"):
        P.validate_variant_grid("1d-sparse", 4, 2)
    with pytest.raises(ValueError, match=r"c\*c to divide p"):
        P.validate_variant_grid("15d-sparse", 6, 2)
    with pytest.raises(ValueError, match="unknown variant"):
        P.validate_variant_grid("2d", 4, 1)
    P.validate_variant_grid("15d-oblivious", 8, 2)


def test_gcn_normalize_bitwise_matches_oracle():
    import distgcn_oracle as O
    rng = np.random.default_rng(3)
    d = np.abs(rng.normal(size=(40, 40))) * (rng.random((40, 40)) < 0.1)
    d[3, 3] = 2.0
    a = P.csr_from_dense(d)
    ours = P.gcn_normalize(a)
    ref = O.gcn_normalize(O.csr_from_dense(d))
    assert np.array_equal(ours.row_ptr, ref.row_ptr)
    assert np.array_equal(ours.col_idx, ref.col_idx)
    assert np.array_equal(ours.values, ref.values)


def test_transpose_and_partition_roundtrip():
    rng = np.random.default_rng(5)
    d = rng.normal(size=(30, 30)) * (rng.random((30, 30)) < 0.2)
    a = P.csr_from_dense(d)
    assert P.csr_equal(P.transpose_csr(P.transpose_csr(a)), a)
    part = P.random_partition(30, 3, seed=4)
    a2, h2 = P.apply_partition(a, np.arange(30.0)[:, None], part)
    assert np.array_equal(a2.to_dense(), d[np.ix_(part.inv_perm, part.inv_perm)])
    assert np.array_equal(h2[:, 0], part.inv_perm.astype(float))


def test_partition_validation_errors():
    with pytest.raises(ValueError):
        P.block_partition(3, 4)
    with pytest.raises(ValueError, match="bijection"):
        P.Partition(3, 1, [0, 0, 0], [0, 0, 1], [(0, 3)])


def test_runtime_generic_p2p_and_deadlock():
    """The generic rank runtime (host payloads) keeps the reference's
    semantics: FIFO per tag, exact charges, deadlock detection."""
    def prog(comm):
        r = comm.rank
        comm.isend((r + 1) % comm.p, np.full(3, float(r)), tag="x")
        got = comm.recv((r - 1) % comm.p, tag="x")
        return got[0]

    res = P.run_program(4, 1, prog)
    assert res.results == [3.0, 0.0, 1.0, 2.0]
    assert res.ledger.counters["p2p"]["data_bytes_sent"].tolist() == [24.0] * 4

    def stuck(comm):
        comm.recv((comm.rank + 1) % comm.p)

    with pytest.raises(P.DeadlockError):
        P.run_program(3, 1, stuck)

    def leftover(comm):
        if comm.rank == 0:
            comm.isend(1, np.zeros(2))

    with pytest.raises(P.SimulationError):
        P.run_program(2, 1, leftover)
