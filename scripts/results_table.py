"""Markdown table of the round's bench lines (profiles/r01/final1, final4)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROWS = [
    ("Reddit-shaped (config 2)", "1 × 1", "final1/reddit_n1.json"),
    ("Reddit-shaped", "2 × 1", "final2/reddit_n2.json"),
    ("Reddit-shaped, 1d-oblivious", "2 × 1", "final2/reddit_n2_obl.json"),
    ("Reddit-shaped", "4 × 1", "final4/reddit_n4.json"),
    ("Reddit-shaped", "4 × 2 (8 ranks)", "final4/reddit_n4_p8.json"),
    ("Reddit-shaped, 15d-sparse c=2", "4 × 2 (8 ranks)", "final4/reddit_n4_p8_15d_c2.json"),
    ("products-shaped (config 3), community layout", "1 × 1", "final1/products_n1.json"),
    ("products-shaped, community partition", "2 × 1", "final2/products_n2.json"),
    ("products-shaped, community partition", "4 × 1", "final4/products_n4.json"),
    ("products-shaped, greedy-tv → GVB", "4 × 1", "final4/products_n4_gvb.json"),
    ("products-shaped, GVB, 1d-oblivious", "4 × 1", "final4/products_n4_gvb_obl.json"),
    ("products-shaped (config 4), GVB, 15d-sparse c=2", "4 × 2 (8 ranks)",
     "final4/products_p8_gvb_15d_c2.json"),
    ("products-shaped (config 4), GVB, 15d-sparse c=4", "4 × 4 (16 ranks)",
     "final4/products_p16_gvb_15d_c4.json"),
    ("papers-shaped (config 5), built in HBM", "4 × 1", "final4/papers_n4.json"),
    ("R-MAT scale 14 (config 1), p=1", "1 × 1", "final1/rmat14_n1.json"),
    ("R-MAT scale 14 (config 1), 4 ranks, 1d-sparse", "1 × 4", "final1/rmat14_p4.json"),
    ("R-MAT scale 14 (config 1), 4 ranks, 1d-oblivious", "1 × 4", "final1/rmat14_p4_obl.json"),
]


def main():
    base = os.path.join(ROOT, "profiles", "r01")
    out = ["| workload | GPUs × ranks | epoch ms | e2e ms | layer-1 SpMM ms (gather TB/s) | "
           "exchange (frac of 775 GB/s) | aware/oblivious volume | file |",
           "|---|---|---|---|---|---|---|---|"]
    for w, g, f in ROWS:
        d = json.loads(open(os.path.join(base, f)).read().strip().splitlines()[-1])
        r = d["roofline"]
        e = d.get("exchange") or {}
        if not e.get("busiest_rank_bytes"):
            e = {}                          # ranks on one GPU: no NVLink traffic
        c = d["comm_elements_per_epoch"]["ratio"]
        k = f"{r['kernel_ms']} ({r['gather_gbs'] / 1000:.1f})" if r.get("kernel_ms") else "—"
        out.append(f"| {w} | {g} | {d['value']} | {(d.get('e2e') or {}).get('value', '—')} | "
                   f"{k} | {e.get('frac', '—')} | {c if c is not None else '—'} | `{f}` |")
    print("\n".join(out))


if __name__ == "__main__":
    sys.exit(main())
