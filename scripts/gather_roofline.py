"""Measure the B200's random-row gather bandwidth (the practical ceiling of
the SpMM's H-row gathers) for row sizes and table footprints matching the
benchmark layers.  Prints one line per case; results go to profiles/."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2504_04673_b200 import _lib as L  # noqa: E402


def main():
    torch.cuda.set_device(0)
    lib = L.lib()
    n_idx = 1 << 24
    out = torch.zeros(4, device="cuda")
    for rows, ld, lanes in [(232965, 16, 4), (232965, 44, 8), (232965, 608, 16),
                            (232965, 608, 32), (232965, 64, 16), (2449029, 16, 4),
                            (2449029, 100, 16), (1 << 22, 64, 16),
                            # 256-bit loads (negative lanes: -lanes lanes x 32 B)
                            (232965, 16, -2), (232965, 64, -8), (232965, 32, -4),
                            (232965, 608, -8)]:
        tab = torch.randn(rows, ld, device="cuda")
        idx = torch.randint(0, rows, (n_idx,), device="cuda", dtype=torch.int32)
        per_group = 64
        lanes_n = abs(lanes)
        groups = 148 * 64 * 8 * 8 // lanes_n * 4
        def go():
            L.check(lib.dg_diag_gather(tab.data_ptr(), ld, idx.data_ptr(), n_idx, lanes, groups,
                                       per_group, out.data_ptr(), L.stream_ptr()))
        go()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 5
        for _ in range(reps):
            go()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps / 1e3
        nbytes = groups * per_group * (lanes_n * 32 if lanes < 0 else lanes * 16)
        foot = rows * ld * 4 / 2**20
        rb = lanes_n * 32 if lanes < 0 else lanes * 16
        print(f"rows={rows} ld={ld} row_bytes={rb} v8={lanes < 0} footprint={foot:.0f}MiB: "
              f"{nbytes / t / 1e9:.0f} GB/s gathered", flush=True)
        del tab, idx


if __name__ == "__main__":
    main()
