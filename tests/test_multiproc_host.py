"""N>1 host-side logic on CPU (gloo, world_size 2): every process builds
the same plan, hosts its block of ranks, charges only those ranks, and the
merged ledger equals the single-process ledger (and the reference's)."""

import os
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, key, q, rank_map="block"):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), DG_RANK_MAP=rank_map)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2504_04673_b200 as P
    from paper_2504_04673_b200.dist import World
    from paper_2504_04673_b200.plan import build_variant_plan, index_setup_charges
    from paper_2504_04673_b200.runtime import CommLedger, ProcessGrid
    from conftest import Golden
    g = Golden("spmm_golden.npz")
    a = g.csr(key + "__a", P.CsrMatrix)
    p, c, vi = (int(x) for x in g[key + "__cfg"])
    variant = P.VARIANTS[vi]
    nb = p // c
    asg = g[key + "__assign"] if nb > 1 else np.zeros(a.n_rows, np.int64)
    sizes = np.bincount(asg, minlength=nb)
    bounds, pos = [], 0
    for s in sizes:
        bounds.append((pos, pos + int(s)))
        pos += int(s)
    part = P.Partition(a.n_rows, nb, asg, g[key + "__perm"], bounds)
    a2, _ = P.apply_partition(a, None, part)
    grid = ProcessGrid(p, c)
    w = World()
    local = w.local_ranks(p)
    dm = P.build_dist_matrices(a2, part.boundaries, grid)
    vp = build_variant_plan(dm.fwd, grid, variant, local)
    full = build_variant_plan(dm.fwd, grid, variant)
    for r in local:      # hosted CSR identical to the full build
        assert np.array_equal(vp.ranks[r].col_ext, full.ranks[r].col_ext)
        assert np.array_equal(vp.ranks[r].row_ptr, full.ranks[r].row_ptr)
    for r in range(p):   # every process knows every halo layout
        assert vp.ranks[r].halo_off == full.ranks[r].halo_off
    led = CommLedger(p, hosted=local)
    index_setup_charges(led, dm.fwd, grid, variant)
    vp.charge(led, g[key + "__h"].shape[1])
    out = [None] * world
    dist.all_gather_object(out, led)
    merged = CommLedger.merged(out)
    ok = all(np.array_equal(merged.counters[pr][nm], ref)
             for (pr, nm), ref in g.ledger_fields(key).items())
    pm = np.array([[s, d, b] for (s, d), b in sorted(merged.pair_max_data_bytes.items())],
                  dtype=np.float64).reshape(-1, 3)
    ok = ok and np.array_equal(pm, g[key + "__pairmax"])
    q.put((rank, ok, local))
    dist.destroy_process_group()


@pytest.mark.parametrize("key,rank_map", [("c7", "block"), ("c8", "block"), ("c12", "block"),
                                          ("c14", "block"), ("c16", "block"), ("c12", "cyclic"),
                                          ("c16", "cyclic")])
def test_two_process_plan_and_ledger(key, rank_map):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + int(key[1:]) * 7 + os.getpid() % 1000 + (3 if rank_map == "cyclic" else 0)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, key, q, rank_map)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    hosted = sorted(r for _, _, loc in res for r in loc)
    assert hosted == sorted(set(hosted))       # disjoint cover of the ranks
    if rank_map == "cyclic":
        for rank, _, loc in res:
            assert all(r % 2 == rank for r in loc)


def _generic_worker(rank, world, port, q):
    """Rank programs using the reference's generic Comm primitives across
    processes (gloo): a ring of isend/recv, all_to_allv and broadcast."""
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import paper_2504_04673_b200 as P
    p = 4

    def program(comm):
        r = comm.rank
        comm.isend((r + 1) % p, np.arange(3, dtype=np.float64) + 10 * r, tag=5)
        comm.isend((r + 2) % p, np.full((2, 2), r, dtype=np.int64), tag="idx")
        got = comm.recv((r - 1) % p, tag=5)
        got2 = comm.recv((r - 2) % p, tag="idx")
        a2a = comm.all_to_allv([np.full(d + 1, 100 * r + d, dtype=np.float64) for d in range(p)])
        b = comm.broadcast(2, np.arange(5, dtype=np.float64) * 7 if r == 2 else None)
        return {"ring": got, "ring2": got2, "a2a": a2a, "b": b}

    run = P.run_program(p, 1, program)
    q.put((rank, run.results, run.ledger.to_dict()))


def test_generic_primitives_across_processes():
    """isend / recv / all_to_allv / broadcast between ranks of different
    processes give the reference's results and ledger (same as one process)."""
    import paper_2504_04673_b200 as P
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29400 + os.getpid() % 1000
    procs = [ctx.Process(target=_generic_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=180) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    p = 4

    def program(comm):
        r = comm.rank
        comm.isend((r + 1) % p, np.arange(3, dtype=np.float64) + 10 * r, tag=5)
        comm.isend((r + 2) % p, np.full((2, 2), r, dtype=np.int64), tag="idx")
        got = comm.recv((r - 1) % p, tag=5)
        got2 = comm.recv((r - 2) % p, tag="idx")
        a2a = comm.all_to_allv([np.full(d + 1, 100 * r + d, dtype=np.float64) for d in range(p)])
        b = comm.broadcast(2, np.arange(5, dtype=np.float64) * 7 if r == 2 else None)
        return {"ring": got, "ring2": got2, "a2a": a2a, "b": b}

    os.environ.pop("WORLD_SIZE", None)
    ref = P.run_program(p, 1, program)
    for _, results, led in res:
        assert led == ref.ledger.to_dict()
        for r in range(p):
            assert np.array_equal(results[r]["ring"], ref.results[r]["ring"])
            assert np.array_equal(results[r]["ring2"], ref.results[r]["ring2"])
            assert np.array_equal(results[r]["b"], ref.results[r]["b"])
            for x, y in zip(results[r]["a2a"], ref.results[r]["a2a"]):
                assert np.array_equal(x, y)
