"""Pin the CPU oracle (oracle/distgcn_oracle.py) to golden vectors produced
by the real reference package (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import distgcn_oracle as O

VARIANTS = O.VARIANTS


def _setup(g, key):
    a = g.csr(key + "__a", O.Csr)
    p, c, vi = (int(x) for x in g[key + "__cfg"])
    return a, p, c, VARIANTS[vi]


def test_spmm_cases_match_reference(spmm_golden):
    g = spmm_golden
    for key in g.cases():
        a, p, c, variant = _setup(g, key)
        asg = g[key + "__assign"]
        nb = p // c
        # the oracle rebuilds the partition from (assignment, perm)
        perm = g[key + "__perm"]
        a2, h2, _ = O.apply_partition(a, g[key + "__h"], perm)
        sizes = np.bincount(asg, minlength=nb)
        bounds, pos = [], 0
        for s in sizes:
            bounds.append((pos, pos + int(s)))
            pos += int(s)
        fwd, _ = O.build_dist_matrices(a2, bounds)
        cols = [fwd["nnz_cols"][(i, j)] for i in range(nb) for j in range(nb)]
        assert np.array_equal([x.size for x in cols], g[key + "__nnzc_len"]), key
        assert np.array_equal(np.concatenate(cols), g[key + "__nnzc"]), key
        led = O.Ledger(p)
        O.exchange_index_lists(led, fwd, p, c, variant)
        hb = [h2[s:e] for s, e in bounds]
        z = O.spmm_all_ranks(led, fwd, hb, p, c, variant)
        z2 = np.vstack([z[i * c] for i in range(nb)])[perm]
        np.testing.assert_allclose(z2, g[key + "__z"], atol=1e-12, rtol=0)
        for (prim, name), ref in g.ledger_fields(key).items():
            assert np.array_equal(led.counters[prim][name], ref), (key, prim, name)
        pm = np.array([[s, d, b] for (s, d), b in sorted(led.pair_max_data_bytes.items())],
                      dtype=np.float64).reshape(-1, 3)
        assert np.array_equal(pm, g[key + "__pairmax"]), key


def test_default_block_partition_run(spmm_golden):
    g = spmm_golden
    for key in g.cases():
        a, p, c, variant = _setup(g, key)
        if not np.array_equal(g[key + "__perm"], np.arange(a.n_rows)):
            continue
        z, led, _, _, _ = O.run_spmm(a, g[key + "__h"], p, c, variant)
        np.testing.assert_allclose(z, g[key + "__z"], atol=1e-12, rtol=0)


def test_gcn_serial_losses_match_reference(gcn_golden):
    g = gcn_golden
    for key in g.cases():
        a = g.csr(key + "__a", O.Csr)
        p, c, layers, hidden, epochs, seed, vi = (int(x) for x in g[key + "__cfg"])
        hist, ws = O.serial_train(a, g[key + "__x"], g[key + "__y"], g[key + "__mask"], layers,
                                  hidden, float(g[key + "__lr"][0]), epochs, seed)
        losses = np.array([h[0] for h in hist])
        # distributed reference runs agree with serial within round-off
        np.testing.assert_allclose(losses, g[key + "__loss"], rtol=0, atol=1e-8)
        for li, w in enumerate(ws):
            np.testing.assert_allclose(w, g[f"{key}__w{li}"], atol=1e-8)


def test_gcn_ledger_matches_reference(gcn_golden):
    g = gcn_golden
    for key in g.cases():
        if key + "__led__p2p__calls" not in g:
            continue
        a = g.csr(key + "__a", O.Csr)
        p, c, layers, hidden, epochs, seed, vi = (int(x) for x in g[key + "__cfg"])
        variant = (VARIANTS + ("serial",))[vi]
        nb = p // c
        perm = g[key + "__perm"]
        a2, _, _ = O.apply_partition(a, None, perm)
        asg = g[key + "__assign"] if nb > 1 else np.zeros(a.n_rows, np.int64)
        sizes = np.bincount(asg, minlength=nb)
        bounds, pos = [], 0
        for s in sizes:
            bounds.append((pos, pos + int(s)))
            pos += int(s)
        fwd, bwd = O.build_dist_matrices(a2, bounds)
        f_out = int(g[key + "__y"].max()) + 1
        dims = O.layer_dims(layers, hidden, g[key + "__x"].shape[1], f_out)
        led = O.train_ledger(fwd, bwd, p, c, variant, epochs, dims)
        for (prim, name), ref in g.ledger_fields(key).items():
            assert np.array_equal(led.counters[prim][name], ref), (key, prim, name)
        for prim in O.PRIMITIVES:
            hist = [led.marks[("epoch", e)][prim]["bytes_sent"] for e in range(epochs)]
            assert np.array_equal(hist, g[f"{key}__hist__{prim}"]), (key, prim)


def test_rmat14_volume_known_answers(rmat_volumes):
    """SURVEY.md A.1 / A.7 numbers, reproduced by the oracle."""
    g = rmat_volumes
    n = 16384
    a = O.Csr(n, n, g["rp"], g["ci"], np.ones(g["ci"].size))
    assert a.nnz == 441602
    led_ref = g.ledger_fields("1d-sparse_4_1")
    # 25,161 rows * 16 * 8 bytes of data in one aware multiply (A.1)
    assert led_ref[("alltoallv", "data_bytes_sent")].sum() == 3_220_608
    assert led_ref[("broadcast", "data_bytes_sent")].sum() == 0
    assert g.ledger_fields("1d-oblivious_4_1")[("broadcast", "data_bytes_sent")].sum() == 6_291_456
    l15 = g.ledger_fields("15d-sparse_8_2")
    assert list(l15[("p2p", "data_bytes_sent")] / 8) == [125968, 0, 100208, 0, 0, 101696, 0,
                                                          74704]
    assert l15[("allreduce", "data_bytes_sent")][0] == 524_288
    # oracle replays the same volumes
    bounds = O.block_boundaries(n, 4)
    fwd, _ = O.build_dist_matrices(a, bounds)
    led = O.Ledger(4)
    O.exchange_index_lists(led, fwd, 4, 1, "1d-sparse")
    O.spmm_all_ranks(led, fwd, [np.zeros((e - s, 16)) for s, e in bounds], 4, 1, "1d-sparse")
    for (prim, name), ref in led_ref.items():
        assert np.array_equal(led.counters[prim][name], ref), (prim, name)
