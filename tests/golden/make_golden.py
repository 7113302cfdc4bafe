"""Generate golden vectors by running the REAL reference package.

Run in the build container only (the reference is not present on the GPU
box):   python tests/golden/make_golden.py
It imports `distgcn` from /root/reference/pkg/src (read-only; nothing is
written there) and writes small .npz fixtures next to this script.  The
fixtures pin both the oracle restatement (tests/test_oracle_golden.py) and
the CUDA path (tests/test_gpu_parity.py).

Inputs are made fp32-representable (adjacency values and features rounded
to float32, then widened) so the float64 reference output is the exact-ish
answer for exactly the inputs the fp32 GPU path sees.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def main():
    sys.path.insert(0, REF)
    from distgcn import graphgen
    from distgcn.gcn import TrainConfig, serial_train, train
    from distgcn.partition import (block_partition, comm_metrics, greedy_tv_partition,
                                   random_partition)
    from distgcn.sparse import CsrMatrix, csr_from_dense, gcn_normalize
    from distgcn.spmm import run_spmm, serial_reference

    def rnd_dense(rng, n, density):
        mask = rng.random((n, n)) < density
        vals = rng.normal(size=(n, n))
        vals[vals == 0.0] = 1.0
        return np.where(mask, vals, 0.0)

    def round_csr(a):
        return CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, f32(a.values))

    def put_csr(out, key, a):
        out[key + "__rp"] = a.row_ptr
        out[key + "__ci"] = a.col_idx
        out[key + "__v"] = a.values
        out[key + "__n"] = np.array([a.n_rows, a.n_cols])

    def put_ledger(out, key, led):
        for prim, c in led.counters.items():
            for name in ("bytes_sent", "data_bytes_sent", "index_bytes_sent",
                         "bytes_received", "data_bytes_received", "msgs_sent",
                         "msgs_received", "calls"):
                out[f"{key}__led__{prim}__{name}"] = np.asarray(c[name])
        pm = sorted(led.pair_max_data_bytes.items())
        out[key + "__pairmax"] = np.array([[s, d, b] for (s, d), b in pm],
                                          dtype=np.float64).reshape(-1, 3)

    # ---------------- SpMM cases ----------------
    spmm = {}
    cases = []
    grid = [("1d-oblivious", 1, 1), ("1d-sparse", 1, 1),
            ("1d-oblivious", 2, 1), ("1d-sparse", 2, 1), ("1d-oblivious", 3, 1),
            ("1d-sparse", 3, 1), ("1d-oblivious", 4, 1), ("1d-sparse", 4, 1),
            ("1d-sparse", 8, 1), ("15d-oblivious", 4, 1), ("15d-sparse", 4, 1),
            ("15d-oblivious", 4, 2), ("15d-sparse", 4, 2), ("15d-oblivious", 8, 2),
            ("15d-sparse", 8, 2), ("15d-sparse", 16, 4), ("15d-oblivious", 16, 4)]
    for ci, (variant, p, c) in enumerate(grid):
        rng = np.random.default_rng(1000 + ci)
        n = int(rng.integers(24, 90))
        f = [1, 3, 4, 16][ci % 4]
        sym = ci % 3 == 0
        d = rnd_dense(rng, n, float(rng.uniform(0.03, 0.2)))
        if sym:
            d = d + d.T
        a = round_csr(csr_from_dense(d))
        h = f32(rng.normal(size=(n, f)))
        part = None
        if ci % 4 == 1 and p // c > 1:
            part = random_partition(n, p // c, seed=ci)
        run = run_spmm(a, h, p, c, variant, partition=part)
        key = f"c{ci}"
        cases.append(key)
        put_csr(spmm, key + "__a", a)
        spmm[key + "__h"] = h
        spmm[key + "__cfg"] = np.array([p, c, ["1d-oblivious", "1d-sparse", "15d-oblivious",
                                               "15d-sparse"].index(variant)])
        spmm[key + "__assign"] = run.partition.assignment
        spmm[key + "__perm"] = run.partition.perm
        spmm[key + "__z"] = run.z
        spmm[key + "__absz"] = serial_reference(
            CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, np.abs(a.values)), np.abs(h))
        put_ledger(spmm, key, run.ledger)
        nb = p // c
        cols = [run.dm.fwd.nnz_cols[(i, j)] for i in range(nb) for j in range(nb)]
        spmm[key + "__nnzc_len"] = np.array([x.size for x in cols], dtype=np.int64)
        spmm[key + "__nnzc"] = (np.concatenate(cols) if cols else np.zeros(0)).astype(np.int64)
        if variant == "1d-sparse" and p > 1:
            m = comm_metrics(a, run.partition, f=f)
            spmm[key + "__send_rows"] = m.per_part_send_rows
    # clique blocks (zero-communication known answer) and an R-MAT-like graph
    a = round_csr(gcn_normalize(graphgen.clique_blocks(4, 6)))
    put_csr(spmm, "clique__a", a)
    spmm["clique__h"] = np.ones((24, 2))
    for v in ("1d-oblivious", "1d-sparse"):
        run = run_spmm(a, spmm["clique__h"], 4, 1, v)
        put_ledger(spmm, f"clique_{v}", run.ledger)
    spmm["cases"] = np.array(cases)
    np.savez_compressed(os.path.join(HERE, "spmm_golden.npz"), **spmm)

    # ---------------- GCN cases ----------------
    gcn = {}
    gcases = []
    setups = [("1d-sparse", 4, 1, 3), ("1d-oblivious", 3, 1, 3), ("15d-sparse", 4, 2, 3),
              ("15d-oblivious", 8, 2, 4), ("1d-sparse", 2, 1, 2), ("serial", 1, 1, 3),
              ("15d-sparse", 4, 1, 3)]
    for gi, (variant, p, c, layers) in enumerate(setups):
        rng = np.random.default_rng(500 + gi)
        n = 48
        if gi == 1:   # directed graph: separate fwd / bwd operands
            d = np.abs(rnd_dense(rng, n, 0.12))
            a_hat = gcn_normalize(csr_from_dense(d))
            feats = rng.normal(size=(n, 5))
            labels = rng.integers(3, size=n)
        else:
            a0, feats, labels = graphgen.sbm(n, blocks=3, seed=gi, feature_dim=5)
            a_hat = gcn_normalize(a0)
        a_hat = round_csr(a_hat)
        feats = f32(feats)
        mask = rng.random(n) < 0.8
        mask[0] = True
        cfg = TrainConfig(layers=layers, hidden=8, lr=0.05, epochs=6, seed=gi + 3,
                          variant=variant)
        part = greedy_tv_partition(a_hat, p // c) if gi == 2 else None
        res = train(a_hat, feats, labels, mask, cfg, p=p, c=c, partition=part)
        key = f"g{gi}"
        gcases.append(key)
        put_csr(gcn, key + "__a", a_hat)
        gcn[key + "__x"] = feats
        gcn[key + "__y"] = labels
        gcn[key + "__mask"] = mask
        gcn[key + "__cfg"] = np.array([p, c, layers, 8, 6, gi + 3,
                                       ["1d-oblivious", "1d-sparse", "15d-oblivious",
                                        "15d-sparse", "serial"].index(variant)])
        gcn[key + "__lr"] = np.array([0.05])
        gcn[key + "__assign"] = (res.partition.assignment if res.partition is not None
                                 else np.zeros(n, np.int64))
        gcn[key + "__perm"] = (res.partition.perm if res.partition is not None
                               else np.arange(n, dtype=np.int64))
        gcn[key + "__loss"] = res.losses
        gcn[key + "__acc"] = np.array([r["train_acc"] for r in res.history])
        for li, w in enumerate(res.weights):
            gcn[f"{key}__w{li}"] = w
        if res.ledger is not None:
            put_ledger(gcn, key, res.ledger)
            for prim in ("p2p", "alltoallv", "broadcast", "allreduce"):
                gcn[f"{key}__hist__{prim}"] = np.array(
                    [r.get(f"{prim}_bytes", 0.0) for r in res.history])
    gcn["cases"] = np.array(gcases)
    np.savez_compressed(os.path.join(HERE, "gcn_golden.npz"), **gcn)

    # ---------------- R-MAT-14 volume known answers -------
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_2504_04673_b200.graphgen import rmat_edges  # scalable input generator
    n, u, v = rmat_edges(14, 16, seed=0)
    rows = np.concatenate([u, v])
    cols = np.concatenate([v, u])
    from distgcn.sparse import csr_from_coo
    a = csr_from_coo(n, n, rows, cols, np.ones(rows.size))
    a.values[:] = 1.0
    a_hat = round_csr(gcn_normalize(a))
    vol_rp, vol_ci = a_hat.row_ptr, a_hat.col_idx
    vol = {"nnz": np.array([a_hat.nnz]), "rp": vol_rp, "ci": vol_ci}
    h = np.zeros((n, 16))
    for variant, p, c in [("1d-sparse", 4, 1), ("1d-oblivious", 4, 1), ("15d-sparse", 8, 2),
                          ("15d-sparse", 16, 4), ("15d-oblivious", 8, 2)]:
        run = run_spmm(a_hat, h, p, c, variant, index_setup=True)
        put_ledger(vol, f"{variant}_{p}_{c}", run.ledger)
    np.savez_compressed(os.path.join(HERE, "rmat14_volumes.npz"), **vol)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()


def make_partition_golden():
    """greedy_tv_partition / volume_balanced_refine assignments from the real
    reference on a few seeded graphs (pins the native partitioners)."""
    sys.path.insert(0, REF)
    from distgcn import graphgen
    from distgcn.partition import greedy_tv_partition, volume_balanced_refine
    from distgcn.sparse import csr_from_dense, gcn_normalize
    out = {}
    graphs = {
        "sbm": graphgen.sbm(120, blocks=4, seed=3)[0],
        "star_aug": graphgen.star_augmented(150, seed=1),
        "grid": graphgen.grid2d(9, 11),
        "directed": None,
    }
    rng = np.random.default_rng(77)
    d = (rng.random((90, 90)) < 0.05).astype(float)
    np.fill_diagonal(d, 0.0)
    graphs["directed"] = csr_from_dense(d)
    keys = []
    for name, a in graphs.items():
        for k, extra in ((3, {}), (4, {"lambda_max": 2.0}), (6, {"epsilon": 0.3})):
            for norm in (False, True):
                a2 = gcn_normalize(a) if norm else a
                tag = f"{name}_k{k}_{int(norm)}"
                g = greedy_tv_partition(a2, k, epsilon=extra.get("epsilon", 0.10))
                v = volume_balanced_refine(a2, g, lambda_max=extra.get("lambda_max"),
                                           epsilon=extra.get("epsilon", 0.10))
                out[tag + "__rp"] = a2.row_ptr
                out[tag + "__ci"] = a2.col_idx
                out[tag + "__v"] = a2.values
                out[tag + "__n"] = np.array([a2.n_rows, a2.n_cols])
                out[tag + "__cfg"] = np.array([k, extra.get("lambda_max", -1.0),
                                               extra.get("epsilon", 0.10)])
                out[tag + "__greedy"] = g.assignment
                out[tag + "__gvb"] = v.assignment
                keys.append(tag)
    out["cases"] = np.array(keys)
    np.savez_compressed(os.path.join(HERE, "partition_golden.npz"), **out)


if __name__ == "__main__":
    make_partition_golden()
