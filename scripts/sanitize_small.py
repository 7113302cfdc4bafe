"""Small end-to-end run touching every kernel (SpMM incl. split rows and
slabs, exchange, group reduce, xent, dense transforms, relu, SGD) for
`compute-sanitizer --tool memcheck` (single process, single GPU)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2504_04673_b200 as P  # noqa: E402
from paper_2504_04673_b200.graphgen import rmat  # noqa: E402


def main():
    a = P.gcn_normalize(rmat(11, 8, 0))
    n = a.n_rows
    rng = np.random.default_rng(0)
    # a hub row longer than the 1024-nonzero chunk: exercises split rows
    rows = np.concatenate([np.zeros(n - 1, np.int64), a.row_of_nnz()])
    cols = np.concatenate([np.arange(1, n), a.col_idx])
    hub = P.csr_from_coo(n, n, rows, cols, np.ones(rows.size))
    for f in (1, 5, 16, 41, 130, 602):
        P.local_spmm(hub, rng.standard_normal((n, f)))
    for variant, p, c in [("1d-sparse", 4, 1), ("1d-oblivious", 3, 1), ("15d-sparse", 8, 2),
                          ("15d-oblivious", 4, 2)]:
        P.run_spmm(a, rng.standard_normal((n, 7)), p, c, variant)
    y = rng.integers(0, 41, size=n)
    x = rng.standard_normal((n, 70))
    for variant, p, c in [("1d-sparse", 2, 1), ("15d-sparse", 4, 2)]:
        for order in ("aggregate-first", "transform-first"):
            P.train(a, x, y, np.ones(n, bool),
                    P.TrainConfig(layers=3, hidden=16, epochs=2, seed=1, variant=variant,
                                  order=order), p=p, c=c)
    print("sanitize run ok")


if __name__ == "__main__":
    main()
