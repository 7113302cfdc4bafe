"""Run under torchrun (one process per GPU): the multi-process CUDA path
against the reference's golden vectors.  Exits non-zero on any mismatch.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/mp_gpu_worker.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2504_04673_b200 as P  # noqa: E402
from conftest import Golden  # noqa: E402
from paper_2504_04673_b200.dist import world  # noqa: E402


def part_of(g, key, n, k):
    asg = g[key + "__assign"] if k > 1 else np.zeros(n, np.int64)
    sizes = np.bincount(asg, minlength=k)
    bounds, pos = [], 0
    for s in sizes:
        bounds.append((pos, pos + int(s)))
        pos += int(s)
    return P.Partition(n, k, asg, g[key + "__perm"], bounds)


def main():
    w = world().init()
    fails = []
    g = Golden("spmm_golden.npz")
    n_checked = 0
    for key in g.cases():
        a = g.csr(key + "__a", P.CsrMatrix)
        p, c, vi = (int(x) for x in g[key + "__cfg"])
        if p < w.size:
            continue
        variant = P.VARIANTS[vi]
        part = part_of(g, key, a.n_rows, p // c)
        run = P.run_spmm(a, g[key + "__h"], p, c, variant, partition=part)
        err = np.abs(run.z - g[key + "__z"])
        if not np.all(err <= 1e-5 * g[key + "__absz"] + 1e-30):
            fails.append((key, "values", float(err.max())))
        for (prim, name), ref in g.ledger_fields(key).items():
            if not np.array_equal(run.ledger.counters[prim][name], ref):
                fails.append((key, prim, name))
        fam = "1d" if variant.startswith("1d") else "15d"
        other = P.run_spmm(a, g[key + "__h"], p, c,
                           f"{fam}-{'oblivious' if variant.endswith('sparse') else 'sparse'}",
                           partition=part)
        if not np.array_equal(other.z, run.z):
            fails.append((key, "aware != oblivious bitwise"))
        n_checked += 1
    gg = Golden("gcn_golden.npz")
    for key in gg.cases():
        a = gg.csr(key + "__a", P.CsrMatrix)
        p, c, layers, hidden, epochs, seed, vi = (int(x) for x in gg[key + "__cfg"])
        variant = (P.VARIANTS + ("serial",))[vi]
        if variant == "serial" or p < w.size:
            continue
        cfg = P.TrainConfig(layers=layers, hidden=hidden, lr=float(gg[key + "__lr"][0]),
                            epochs=epochs, seed=seed, variant=variant)
        part = part_of(gg, key, a.n_rows, p // c) if p // c > 1 else None
        res = P.train(a, gg[key + "__x"], gg[key + "__y"], gg[key + "__mask"], cfg, p=p, c=c,
                      partition=part)
        if not np.allclose(res.losses, gg[key + "__loss"], rtol=1e-5, atol=0):
            fails.append((key, "loss", res.losses.tolist()))
        for (prim, name), ref in gg.ledger_fields(key).items():
            if not np.array_equal(res.ledger.counters[prim][name], ref):
                fails.append((key, "gcn ledger", prim, name))
        for per_rank in res.weights_per_rank[1:]:
            for w0, wr in zip(res.weights_per_rank[0], per_rank):
                if not np.array_equal(w0, wr):
                    fails.append((key, "replication"))
        n_checked += 1
        if variant.startswith("15d") and c > 1:   # extension: post-transform reduction
            import dataclasses
            res2 = P.train(a, gg[key + "__x"], gg[key + "__y"], gg[key + "__mask"],
                           dataclasses.replace(cfg, reduce_after_transform=True), p=p, c=c,
                           partition=part)
            if not np.allclose(res2.losses, gg[key + "__loss"], rtol=1e-5, atol=0):
                fails.append((key, "reduce_after_transform loss", res2.losses.tolist()))
            for per_rank in res2.weights_per_rank[1:]:
                for w0, wr in zip(res2.weights_per_rank[0], per_rank):
                    if not np.array_equal(w0, wr):
                        fails.append((key, "reduce_after_transform replication"))
            n_checked += 1
    # HBM-resident sharded path (sharded.py): each process builds only its
    # block rows; single-buffered halos; must equal the host-plan GcnRun
    import torch
    from paper_2504_04673_b200 import graphgen, sharded
    a = P.gcn_normalize(graphgen.rmat(11, 8, 5))
    a.values = a.values.astype(np.float32).astype(np.float64)
    for p in sorted({w.size, 2 * w.size}):
        f_in, classes = 40, 9
        cfg = P.TrainConfig(layers=3, hidden=16, lr=0.1, epochs=3, seed=2, variant="1d-sparse")
        sg = sharded.ShardedGraph.from_csr(a, p)
        x, y = sharded.sharded_inputs(sg, f_in, classes, seed=4)
        gr = sharded.sharded_gcn_run(sg, x, y, f_in, classes, cfg)
        res = gr.result(gr.run())
        gr.close()
        # host reference: the full inputs, assembled from every process's blocks
        xs = w.all_gather_object({i: t[:, :f_in].cpu().numpy() for i, t in x.items()})
        ys = w.all_gather_object({i: t.cpu().numpy() for i, t in y.items()})
        xd, yd = {}, {}
        for d in xs:
            xd.update(d)
        for d in ys:
            yd.update(d)
        xf = np.concatenate([xd[i] for i in range(p)])
        yf = np.concatenate([yd[i] for i in range(p)])
        ref = P.train(a, xf, yf, np.ones(a.n_rows, bool), cfg, p=p)
        if not np.array_equal(res.losses, ref.losses):
            fails.append(("sharded", p, "loss", res.losses.tolist(), ref.losses.tolist()))
        for w1, w2 in zip(res.weights, ref.weights):
            if not np.array_equal(w1, w2):
                fails.append(("sharded", p, "weights"))
        for prim in ref.ledger.counters:
            for name, v in ref.ledger.counters[prim].items():
                if not np.array_equal(res.ledger.counters[prim][name], v):
                    fails.append(("sharded", p, "ledger", prim, name))
        n_checked += 1
        del x, y, sg
        torch.cuda.empty_cache()
    # gather-free runs: the device-side global loss equals the gathered one
    from paper_2504_04673_b200.gcn import GcnRun
    a = P.gcn_normalize(graphgen.rmat(10, 8, 6))
    rng = np.random.default_rng(3)
    x = rng.standard_normal((a.n_rows, 20)).astype(np.float32)
    yv = rng.integers(0, 6, a.n_rows)
    cfg = P.TrainConfig(layers=3, hidden=16, lr=0.1, epochs=2, seed=3)
    for p in sorted({w.size, 2 * w.size}):
        gr = GcnRun(a, x, yv, np.ones(a.n_rows, bool), cfg, p=p)
        full = gr.result(gr.run())
        tot = gr.global_stats(gr.run(gather=False)).cpu().numpy()
        losses = tot[:, 0] / a.n_rows
        if not np.allclose(losses, full.losses, rtol=1e-6, atol=0):
            fails.append(("global_stats", p, losses.tolist(), full.losses.tolist()))
        gr.close()
        n_checked += 1
    # lock-step host driver (several ranks per process) == thread-per-rank runtime
    for p, c, variant in [(2 * w.size, 1, "1d-sparse"), (4 * w.size, 2, "15d-sparse")]:
        if variant.startswith("15d") and p % (c * c):
            continue
        cfg = P.TrainConfig(layers=3, hidden=16, lr=0.1, epochs=2, seed=3, variant=variant)
        gr = GcnRun(a, x, yv, np.ones(a.n_rows, bool), cfg, p=p, c=c)
        ref = gr.result(gr.run())
        got = gr.result(gr.run_lockstep())
        if not np.array_equal(got.losses, ref.losses):
            fails.append(("lockstep", p, c, got.losses.tolist(), ref.losses.tolist()))
        for w1, w2 in zip(got.weights_per_rank, ref.weights_per_rank):
            for a1, a2 in zip(w1, w2):
                if not np.array_equal(a1, a2):
                    fails.append(("lockstep weights", p, c))
        for prim in ref.ledger.counters:
            for name, v in ref.ledger.counters[prim].items():
                if not np.array_equal(got.ledger.counters[prim][name], v):
                    fails.append(("lockstep ledger", p, c, prim, name))
        gr.close()
        n_checked += 1
    print(f"[proc {w.proc}/{w.size}] checked {n_checked} cases, {len(fails)} failures",
          flush=True)
    for f in fails:
        print("FAIL", f, flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
