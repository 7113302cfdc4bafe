"""Seeded, scalable synthetic graphs for tests and the benchmark.

The reference's generators (graphgen.py:26-120) build an n x n dense draw
(O(n^2) memory) and have no R-MAT; the benchmark configs (BASELINE.json
configs 1-5) name R-MAT and Reddit/products-shaped power-law graphs, so
these generators are new: vectorised NumPy, O(edges) memory.

All return symmetric unit-weight adjacency without self-loops, as the
reference generators do (graphgen.py:18-23: duplicates collapse to 1.0);
`gcn_normalize` adds the self-loops.
"""

from __future__ import annotations

import numpy as np

from .sparse import CsrMatrix

__all__ = ["rmat_edges", "rmat", "reddit_shaped", "products_shaped", "symmetric_unit",
           "gaussian_features", "clique_blocks", "sbm", "planted_partition", "chung_lu_host"]

GRAPH500 = (0.57, 0.19, 0.19)


def rmat_edges(scale, edge_factor=16, seed=0, m=None, abc=GRAPH500, rng=None):
    """R-MAT pairs (u, v) over 2^scale vertices, one uniform draw per bit
    level, least significant bit first -- the SURVEY.md Appendix A recipe
    (reproduces its R-MAT-14 probe numbers exactly: 441,602 stored
    nonzeros after normalisation, p=4 send rows [7873, 6263, 6356, 4669]).
    Self-loops are dropped.  Returns (n, u, v) as int64 arrays."""
    a, b, c = abc
    n = 1 << scale
    m = edge_factor * n if m is None else int(m)
    rng = np.random.default_rng(seed) if rng is None else rng
    u = np.zeros(m, dtype=np.int64)
    v = np.zeros(m, dtype=np.int64)
    for level in range(scale):
        r = rng.random(m)
        bit = np.int64(1) << np.int64(level)
        down = r >= a + b            # quadrants c, d set the row bit
        right = ((r >= a) & (r < a + b)) | (r >= a + b + c)
        u += np.where(down, bit, 0)
        v += np.where(right, bit, 0)
    keep = u != v
    return n, u[keep], v[keep]


def symmetric_unit(n, u, v) -> CsrMatrix:
    """Symmetric 0/1 adjacency from pairs: mirror, dedup, drop self-loops,
    canonical CSR (ascending columns)."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    keep = u != v
    u, v = u[keep], v[keep]
    key = np.unique(np.concatenate([u * n + v, v * n + u]))
    rows, cols = key // n, key % n
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
    return CsrMatrix(n, n, rp, cols, np.ones(cols.size), check=False)


def rmat(scale, edge_factor=16, seed=0) -> CsrMatrix:
    """Config 1 graph: Graph500 R-MAT, symmetrised, unit weights."""
    n, u, v = rmat_edges(scale, edge_factor, seed)
    return symmetric_unit(n, u, v)


def _rmat_target(n, target_nnz, seed, abc):
    """R-MAT on the next power of two with ids >= n rejected, sampled in
    rounds until the symmetric pattern holds >= target_nnz stored
    off-diagonal entries, then trimmed (seeded) to exactly target_nnz/2
    undirected pairs."""
    scale = int(np.ceil(np.log2(n)))
    rng = np.random.default_rng(seed)
    want = target_nnz // 2
    keys = np.zeros(0, dtype=np.int64)
    m = int(want * 1.3)
    while keys.size < want:
        _, u, v = rmat_edges(scale, m=m, abc=abc, rng=rng)
        ok = (u < n) & (v < n)
        u, v = u[ok], v[ok]
        lo, hi = np.minimum(u, v), np.maximum(u, v)
        keys = np.unique(np.concatenate([keys, lo * n + hi]))
        m = int(max(want - keys.size, 1) * 1.6) + 1024
    if keys.size > want:
        keys = np.sort(rng.choice(keys, size=want, replace=False))
    return symmetric_unit(n, keys // n, keys % n)


def reddit_shaped(n=232_965, nnz=114_848_857, seed=0, abc=GRAPH500) -> CsrMatrix:
    """Config 2: Reddit-shaped power-law graph (PAPER.md:547 counts 114.8M
    stored nonzeros).  `nnz` counts stored off-diagonal entries (both
    directions); gcn_normalize adds n self-loops."""
    return _rmat_target(n, nnz - (nnz % 2), seed, abc)


def planted_partition(n, nnz, k=64, p_in=0.8, seed=0, abc=GRAPH500) -> CsrMatrix:
    """Power-law planted partition: an R-MAT degree skew inside k hidden
    communities (fraction p_in of edges intra-community), with the
    community structure hidden by a seeded random relabel."""
    rng = np.random.default_rng(seed)
    want = nnz // 2
    size = -(-n // k)
    scale_in = int(np.ceil(np.log2(size)))
    scale_all = int(np.ceil(np.log2(n)))
    keys = np.zeros(0, dtype=np.int64)
    relabel = rng.permutation(n).astype(np.int64)
    while keys.size < want:
        need = want - keys.size
        m_in = int(need * p_in * 1.4) + 1024
        m_out = int(need * (1 - p_in) * 1.4) + 1024
        _, u, v = rmat_edges(scale_in, m=m_in, abc=abc, rng=rng)
        comm = rng.integers(0, k, size=u.size)
        u, v = u + comm * size, v + comm * size
        _, u2, v2 = rmat_edges(scale_all, m=m_out, abc=abc, rng=rng)
        u = np.concatenate([u, u2])
        v = np.concatenate([v, v2])
        ok = (u < n) & (v < n) & (u != v)
        u, v = relabel[u[ok]], relabel[v[ok]]
        lo, hi = np.minimum(u, v), np.maximum(u, v)
        keys = np.unique(np.concatenate([keys, lo * n + hi]))
    if keys.size > want:
        keys = np.sort(rng.choice(keys, size=want, replace=False))
    return symmetric_unit(n, keys // n, keys % n)


def products_shaped(n=2_449_029, nnz=2 * 61_859_140, seed=0) -> CsrMatrix:
    """Config 3/4: ogbn-products-shaped planted-partition power-law graph."""
    return planted_partition(n, nnz, k=64, seed=seed)


def gaussian_features(n, dim, seed=0, dtype=np.float32) -> np.ndarray:
    """N(0,1) features; float32 by default (the GPU path's input type)."""
    return np.random.default_rng(seed).standard_normal((n, dim)).astype(dtype)


def clique_blocks(num_cliques, size) -> CsrMatrix:
    """Disjoint cliques (block-diagonal pattern), like graphgen.py:75-85."""
    n = num_cliques * size
    i, j = np.meshgrid(np.arange(size), np.arange(size), indexing="ij")
    off = (i != j)
    base = np.arange(num_cliques)[:, None] * size
    uu = (base + i[off].ravel()[None, :]).ravel()
    vv = (base + j[off].ravel()[None, :]).ravel()
    return symmetric_unit(n, uu, vv)


def sbm(n, blocks=2, p_in=0.2, p_out=0.01, seed=0, feature_dim=16, feature_scale=2.0,
        noise=1.0):
    """Stochastic block model with label-informative features; same draw
    sequence as the reference (graphgen.py:26-49) so small instances agree."""
    rng = np.random.default_rng(seed)
    base, rem = divmod(n, blocks)
    sizes = [base + 1] * rem + [base] * (blocks - rem)
    labels = np.repeat(np.arange(blocks, dtype=np.int64), sizes)
    prob = np.where(labels[:, None] == labels[None, :], p_in, p_out)
    draw = rng.random((n, n))
    rows, cols = np.nonzero(np.triu(draw < prob, k=1))
    a = symmetric_unit(n, rows, cols)
    means = rng.normal(size=(blocks, feature_dim)) * feature_scale
    features = means[labels] + rng.normal(size=(n, feature_dim)) * noise
    return a, features, labels


# ---------------------------------------------------------------------------
# large shaped graphs, generated on the GPU (benchmark input synthesis)
# ---------------------------------------------------------------------------

def _host_cumsum(t):
    import torch
    return torch.from_numpy(np.cumsum(t.cpu().numpy())).to(t.device)


def chung_lu_device(n, pairs, alpha=0.6, max_weight=None, seed=0, communities=0, p_in=0.8,
                    return_communities=False, device=None):
    """Power-law (Chung-Lu) symmetric 0/1 graph with exactly `pairs`
    undirected edges, sampled on the GPU with torch (input synthesis only).

    Expected degree of vertex of rank k ~ (k+1)^-alpha, capped at
    `max_weight`, then a seeded random relabel so hubs are scattered.  With
    `communities` > 0 a fraction p_in of the edges is drawn inside hidden
    equal-size communities (planted partition, products-shaped).
    Returns a host CsrMatrix (int64 indices, unit values).  `device`
    (default: the current CUDA device) only decides where the draws run;
    tests use a CPU device for small instances."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    w = (torch.arange(n, device=dev, dtype=torch.float64) + 1.0) ** (-alpha)
    w = w / w.sum() * (2.0 * pairs)
    if max_weight is not None:
        for _ in range(8):
            w = torch.clamp(w, max=float(max_weight))
            w = w / w.sum() * (2.0 * pairs)
    w = w[torch.randperm(n, generator=g, device=dev)]
    # CDFs by a sequential host sum: a parallel GPU scan's float association
    # depends on timing, and under torchrun every process must draw the
    # identical graph
    cdf = _host_cumsum(w)
    cdf = cdf / cdf[-1]
    if communities:
        comm = torch.randint(0, communities, (n,), generator=g, device=dev)
        order = torch.argsort(comm, stable=True)
        cstart = torch.searchsorted(comm[order], torch.arange(communities + 1, device=dev))
        wc = w[order]
        ccdf = _host_cumsum(wc)
    keys = torch.zeros(0, dtype=torch.int64, device=dev)
    while keys.numel() < pairs:
        m = int((pairs - keys.numel()) * 1.3) + 4096
        u = torch.searchsorted(cdf, torch.rand(m, generator=g, device=dev, dtype=torch.float64))
        if communities:
            # partner inside u's community for a fraction p_in of the draws
            cu = comm[torch.clamp(u, max=n - 1)]
            lo_c, hi_c = cstart[cu], cstart[cu + 1]
            base = torch.where(lo_c > 0, ccdf[torch.clamp(lo_c - 1, min=0)],
                               torch.zeros_like(ccdf[0:1]).expand_as(lo_c))
            span = ccdf[hi_c - 1] - base
            r = base + torch.rand(m, generator=g, device=dev, dtype=torch.float64) * span
            vin = order[torch.clamp(torch.searchsorted(ccdf, r), max=n - 1)]
            vout = torch.searchsorted(cdf, torch.rand(m, generator=g, device=dev,
                                                      dtype=torch.float64))
            pick = torch.rand(m, generator=g, device=dev) < p_in
            v = torch.where(pick, vin, vout)
        else:
            v = torch.searchsorted(cdf, torch.rand(m, generator=g, device=dev,
                                                   dtype=torch.float64))
        u = torch.clamp(u, max=n - 1)
        v = torch.clamp(v, max=n - 1)
        ok = u != v
        u, v = u[ok], v[ok]
        k = torch.minimum(u, v) * n + torch.maximum(u, v)
        keys = torch.unique(torch.cat([keys, k]))
    if keys.numel() > pairs:
        keys = keys[torch.randperm(keys.numel(), generator=g, device=dev)[:pairs]]
    lo, hi = keys // n, keys % n
    rows = torch.cat([lo, hi])
    cols = torch.cat([hi, lo])
    key2, _ = torch.sort(rows * n + cols)
    rows, cols = key2 // n, key2 % n
    rp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    rp[1:] = torch.cumsum(torch.bincount(rows, minlength=n), 0)
    out = CsrMatrix(n, n, rp.cpu().numpy(), cols.cpu().numpy(), np.ones(cols.numel()),
                    check=False)
    comm_host = comm.cpu().numpy() if communities else None
    del keys, rows, cols, key2, rp
    if dev.type == "cuda":
        torch.cuda.empty_cache()
    return (out, comm_host) if return_communities else out


def chung_lu_host(n, pairs, alpha=0.6, max_weight=None, seed=0) -> CsrMatrix:
    """Host (NumPy) Chung-Lu graph with exactly `pairs` undirected edges and
    the same degree law as `chung_lu_device` (rank-k weight ~ (k+1)^-alpha,
    capped, randomly relabelled).  Used for the CPU reference arm's
    scaled-down samples of configs 2, 3 and 5 (same average degree), where
    no device may be involved."""
    rng = np.random.default_rng(seed)
    w = (np.arange(n, dtype=np.float64) + 1.0) ** (-alpha)
    w = w / w.sum() * (2.0 * pairs)
    if max_weight is not None:
        for _ in range(8):
            w = np.minimum(w, float(max_weight))
            w = w / w.sum() * (2.0 * pairs)
    w = w[rng.permutation(n)]
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    keys = np.zeros(0, dtype=np.int64)
    while keys.size < pairs:
        m = int((pairs - keys.size) * 1.3) + 4096
        u = np.minimum(np.searchsorted(cdf, rng.random(m)), n - 1)
        v = np.minimum(np.searchsorted(cdf, rng.random(m)), n - 1)
        ok = u != v
        u, v = u[ok], v[ok]
        keys = np.unique(np.concatenate([keys, np.minimum(u, v) * n + np.maximum(u, v)]))
    if keys.size > pairs:
        keys = np.sort(rng.choice(keys, size=pairs, replace=False))
    return symmetric_unit(n, keys // n, keys % n)


def reddit_shaped_device(seed=0, n=232_965, nnz=114_848_856):
    """Config 2 graph on the GPU: 232,965 vertices, 114.8M stored
    off-diagonal nonzeros, power-law degrees capped near
    Reddit's maximum degree (21,657)."""
    return chung_lu_device(n, nnz // 2, alpha=0.6, max_weight=21_657, seed=seed)


def products_shaped_device(seed=0, n=2_449_029, nnz=2 * 61_859_140, communities=256,
                           p_in=0.8):
    """Config 3/4 graph on the GPU: 2.45M vertices, 123.7M stored
    off-diagonal nonzeros, power-law degrees inside hidden communities
    (a fraction p_in of the edges inside them).
    Returns (adjacency, planted community of every vertex)."""
    return chung_lu_device(n, nnz // 2, alpha=0.55, max_weight=17_481, seed=seed,
                           communities=communities, p_in=p_in, return_communities=True)


# ---------------------------------------------------------------------------
# the reference's small generators (graphgen.py:52-120), same draw sequences
# ---------------------------------------------------------------------------

def grid2d(rows, cols) -> CsrMatrix:
    """4-neighbour lattice, row-major numbering (graphgen.py:52-65)."""
    idx = np.arange(rows * cols, dtype=np.int64).reshape(rows, cols)
    u = np.concatenate([idx[:, :-1].ravel(), idx[:-1, :].ravel()])
    v = np.concatenate([idx[:, 1:].ravel(), idx[1:, :].ravel()])
    return symmetric_unit(rows * cols, u, v)


def star(leaves) -> CsrMatrix:
    """Vertex 0 joined to `leaves` leaves (graphgen.py:68-72)."""
    return symmetric_unit(leaves + 1, np.zeros(leaves, np.int64),
                          np.arange(1, leaves + 1, dtype=np.int64))


def star_augmented(n, seed=0, community_fracs=(0.35, 0.25, 0.2, 0.12, 0.08), avg_degree=8.0,
                   p_out=0.002, hubs=3, hub_frac=0.15) -> CsrMatrix:
    """Unequal communities plus global hubs (graphgen.py:88-120)."""
    rng = np.random.default_rng(seed)
    sizes = [max(2, int(round(f * n))) for f in community_fracs]
    sizes[-1] = n - sum(sizes[:-1])
    if sizes[-1] < 2:
        raise ValueError("n too small for the community layout")
    labels = np.repeat(np.arange(len(sizes)), sizes)
    p_in = np.minimum(avg_degree / np.maximum(np.array(sizes) - 1, 1), 1.0)
    prob = np.where(labels[:, None] == labels[None, :], p_in[labels][:, None], p_out)
    draw = rng.random((n, n))
    rows, cols = np.nonzero(np.triu(draw < prob, k=1))
    starts = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    hr, hc = [rows], [cols]
    for h in range(min(hubs, len(sizes))):
        hub = int(starts[h])
        targets = rng.choice(n, size=max(1, int(hub_frac * n)), replace=False)
        targets = targets[targets != hub]
        hr.append(np.full(targets.size, hub, dtype=np.int64))
        hc.append(targets.astype(np.int64))
    return symmetric_unit(n, np.concatenate(hr), np.concatenate(hc))
