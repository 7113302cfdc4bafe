"""Label propagation at products scale: communities found vs the planted
ones (generator labels are used here only to grade the result)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_04673_b200 import graphgen  # noqa: E402
from paper_2504_04673_b200.locality import _edges, label_propagation  # noqa: E402

torch.cuda.set_device(0)
a, comm = graphgen.products_shaped_device(seed=0)
dev = torch.device("cuda", 0)
rows, cols = _edges(a.row_ptr, a.col_idx, a.n_rows, dev)
for iters in (4, 8, 12, 20):
    torch.cuda.synchronize()
    t = time.time()
    lab = label_propagation(rows, cols, a.n_rows, iters=iters)
    torch.cuda.synchronize()
    dt = time.time() - t
    l = lab.cpu().numpy()
    u, cnt = np.unique(l, return_counts=True)
    r, c = rows.cpu().numpy(), cols.cpu().numpy()
    intra = (l[r] == l[c]).mean()
    top = u[np.argsort(-cnt)[:300]]
    pure = sum(np.bincount(comm[l == x]).max() for x in top)
    print(f"iters={iters} {dt:.2f}s labels={u.size} largest={np.sort(cnt)[-5:].tolist()} "
          f"smallest={np.sort(cnt)[:5].tolist()} intra-label edges={intra:.3f} "
          f"(planted {(comm[r] == comm[c]).mean():.3f}) "
          f"purity(top300)={pure / np.sort(cnt)[-300:].sum():.3f}", flush=True)
