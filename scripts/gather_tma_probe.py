"""Random-row gather bandwidth through TMA tile::gather4 (probe.cu) next to
the 256-bit register-path probe (dg_diag_gather) on the same tables: does
TMA feed indexed row gathers faster than LDG on B200?  One line per case."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2504_04673_b200 import _lib as L  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def main():
    torch.cuda.set_device(0)
    lib = L.lib()
    n_idx = 1 << 24
    out = torch.zeros(4, device="cuda")
    cases = [  # rows, ld, box, [(variant, ctas)], ldg lanes (-: 256-bit)
        (232965, 608, 64, [(0, 148), (1, 148), (2, 296), (3, 296)], -8),
        (232965, 64, 64, [(0, 148), (2, 296)], -8),
        (232965, 608, 128, [(0, 148), (2, 296)], -16),
        (2449029, 16, 16, [(0, 296), (2, 296), (2, 592)], -2),
        (2449029, 128, 128, [(0, 148), (2, 296)], -16),
    ]
    for rows, ld, box, tv, lanes in cases:
        tab = torch.randn(rows, ld, device="cuda")
        idx = torch.randint(0, rows, (n_idx,), device="cuda", dtype=torch.int32)
        nbytes = n_idx * box * 4
        foot = rows * ld * 4 / 2**20
        for var, ctas in tv:
            t = timed(lambda: L.check(lib.dg_diag_gather_tma(
                tab.data_ptr(), ld, rows, 0, box, idx.data_ptr(), n_idx, var, ctas,
                out.data_ptr(), L.stream_ptr())))
            print(f"TMA gather4 rows={rows} ld={ld} box={box} ({box * 4} B rows) "
                  f"footprint={foot:.0f}MiB variant={var} ctas={ctas}: "
                  f"{nbytes / t / 1e9:.0f} GB/s", flush=True)
        ln = abs(lanes)
        per_group = 64
        groups = n_idx // per_group
        t = timed(lambda: L.check(lib.dg_diag_gather(tab.data_ptr(), ld, idx.data_ptr(), n_idx,
                                                     lanes, groups, per_group, out.data_ptr(),
                                                     L.stream_ptr())))
        rb = ln * 32
        print(f"LDG.256  rows={rows} ld={ld} row_bytes={rb} footprint={foot:.0f}MiB: "
              f"{groups * per_group * rb / t / 1e9:.0f} GB/s", flush=True)
        del tab, idx


if __name__ == "__main__":
    main()
