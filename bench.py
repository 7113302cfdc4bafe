"""Benchmark: GCN epoch time + SpMM HBM GB/s + comm bytes vs oblivious.

Metric (BASELINE.json): "GCN epoch ms & SpMM HBM GB/s at 1/2/4/8 B200; comm
bytes vs oblivious".  At N=1 the workload is config 2 (Reddit-shaped graph,
232,965 vertices, 114.8M stored nonzeros + self-loops, f_in=602, 2-layer GCN
= TrainConfig(layers=3, hidden=16), C=41 classes, 1D sparsity-aware SpMM).
A "step" is one full training epoch (forward + backward + SGD) over the
whole graph.  `value` = ms per epoch (lower is better).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU algorithm (the NumPy oracle
port, oracle/distgcn_oracle.py, same np.add.at hot loop as
sparse.py:222) on a bounded sample of the same workload and extrapolates
the full-epoch time from its measured nnz*f throughput.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
if "papers" in sys.argv:
    # config 5 fills HBM: avoid caching-allocator fragmentation (our IPC
    # buffers are cudaMalloc'd by the library, not by torch)
    os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0

WORKLOADS = {
    "reddit": dict(desc="Reddit-shaped power-law graph (232,965 vertices, 114,848,856 stored "
                        "off-diagonal nonzeros + 232,965 self-loops), f_in=602, 2-layer GCN "
                        "(layers=3, hidden=16), C=41",
                   n=232_965, f_in=602, classes=41, layers=3, hidden=16),
    "rmat14": dict(desc="R-MAT scale 14 (Graph500 .57/.19/.19, edge factor 16), f=16, "
                        "2-layer GCN (layers=3, hidden=16), C=16",
                   n=16_384, f_in=16, classes=16, layers=3, hidden=16),
    "products": dict(desc="ogbn-products-shaped planted-partition power-law graph (2,449,029 "
                          "vertices, 123,718,280 stored off-diagonal nonzeros + self-loops, 256 "
                          "hidden communities), f_in=100, 3-layer GCN (layers=4, hidden=16), C=47, "
                          "community-preserving partition",
                     n=2_449_029, f_in=100, classes=47, layers=4, hidden=16),
    "papers": dict(desc="ogbn-papers100M-shaped power-law graph (111,059,956 vertices, ~3.23B "
                        "stored off-diagonal nonzeros + self-loops, Chung-Lu alpha=0.7, degree cap "
                        "30,000), f_in=128, 3-layer GCN (layers=4, hidden=16), C=172, block "
                        "partition, built sharded in HBM (sharded.py)",
                   n=111_059_956, f_in=128, classes=172, layers=4, hidden=16),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


TRAFFIC = os.path.join(ROOT, "profiles", "traffic.json")


def ncu_traffic(key):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the
    dominant kernel, from the committed `ncu --set full` capture
    (profiles/traffic.json, written by scripts/ncu_traffic.py)."""
    try:
        with open(TRAFFIC) as fh:
            return json.load(fh).get(key)
    except Exception:  # noqa: BLE001
        return None


def nvlink_peak():
    """Measured peer-copy GB/s per direction (profiles/nvlink.json, written
    from scripts/nvlink_probe.py), else the B200_PROFILING.md figure."""
    try:
        with open(os.path.join(ROOT, "profiles", "nvlink.json")) as fh:
            return float(json.load(fh)["peer_copy_gbs"]), "measured (profiles/nvlink.json)"
    except Exception:  # noqa: BLE001
        return 770.0, "B200_PROFILING.md measured peer copy"


def gather_probe(rows, ld):
    """Measured pure-gather rate (random 256-B row slabs, 256-bit loads, no
    CSR, no math) for this table geometry, from profiles/r01/
    gather_roofline_v8.txt (scripts/gather_roofline.py), or None."""
    import re
    try:
        with open(os.path.join(ROOT, "profiles", "r01", "gather_roofline_v8.txt")) as fh:
            for line in fh:
                m = re.match(r"rows=(\d+) ld=(\d+) row_bytes=256 v8=True .*: (\d+) GB/s", line)
                if m and int(m.group(1)) == rows and int(m.group(2)) == ld:
                    return float(m.group(3))
    except OSError:
        pass
    return None


def peaks():
    try:
        with open(PEAKS) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"




def make_graph(name, seed=0, p_in=0.8):
    import paper_2504_04673_b200 as P
    from paper_2504_04673_b200 import graphgen
    t = time.time()
    if name == "reddit":
        a = graphgen.reddit_shaped_device(seed=seed)
    elif name == "products":
        a, _ = graphgen.products_shaped_device(seed=seed, p_in=p_in)  # planted labels unused
    else:
        a = graphgen.rmat(14, 16, seed)
    log(f"[bench] graph {name}: n={a.n_rows} nnz={a.nnz} ({time.time() - t:.1f}s)")
    t = time.time()
    ah = P.gcn_normalize(a)
    # fp32-representable values: the GPU path and the CPU reference see the same numbers
    ah.values = ah.values.astype(np.float32).astype(np.float64)
    log(f"[bench] gcn_normalize: nnz={ah.nnz} ({time.time() - t:.1f}s)")
    return ah


def make_inputs(wl, n, seed=1):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, wl["f_in"]), dtype=np.float32)
    y = np.random.default_rng(2).integers(0, wl["classes"], size=n)
    mask = np.ones(n, dtype=bool)
    return x, y, mask


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: NVML queried from a background thread every 2 ms (so even a
    12 ms timed region of config 1 gets samples), one sample at start and at
    stop; nvidia-smi polling (100 ms) when NVML is unavailable."""

    _REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                "sw_power_cap": 0x4}

    def __init__(self, gpu=0, period_s=0.002):
        import threading
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.p = None
        self._stop = threading.Event()
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = self._handle(N, gpu)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
            self._sample()
            self.t = threading.Thread(target=self._loop, args=(period_s,), daemon=True)
            self.t.start()
            self.source = "nvml (2 ms)"
        except Exception:  # noqa: BLE001 - fall back to nvidia-smi polling
            self.N = None
            self._start_smi(gpu)

    @staticmethod
    def _handle(N, gpu):
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(gpu).uuid)
            return N.nvmlDeviceGetHandleByUUID(("GPU-" + uuid).encode())
        except Exception:  # noqa: BLE001
            return N.nvmlDeviceGetHandleByIndex(gpu)

    def _sample(self):
        N = self.N
        self.samples.append(float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)))
        try:
            mask = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except AttributeError:
            mask = N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        for name, bit in self._REASONS.items():
            if mask & bit:
                self.reasons.add(name)

    def _loop(self, period):
        while not self._stop.wait(period):
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                return

    def _start_smi(self, gpu):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        self.source = "nvidia-smi (100 ms)"
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.p = None

    def stop(self):
        if self.N is not None:
            self._stop.set()
            self.t.join()
            self._sample()
            sm = self.samples
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(self.reasons), "samples": len(sm),
                    "sm_mhz_min": min(sm), "source": self.source}
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "source": self.source}


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the oracle port on a bounded sample
# ---------------------------------------------------------------------------

def cpu_reference_epoch_ms(a_hat, wl, budget_s=20.0, nnz_total=None):
    """Time the reference's CPU hot loop (np.add.at local_spmm, sparse.py:222,
    via the oracle port) on row samples of the same graph at each SpMM
    width of the epoch, then extrapolate the full epoch:
    sum over the 2(L-1) multiply phases of nnz*f / measured rate.  The
    GEMMs / loss are not timed (<6% of the reference's epoch)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import distgcn_oracle as O
    dims = [wl["f_in"]] + [wl["hidden"]] * (wl["layers"] - 2) + [wl["classes"]]
    widths = dims[:-1] + dims[1:]           # forward widths, then backward widths
    nnz_total = a_hat.nnz if nnz_total is None else int(nnz_total)
    rates = {}
    per_width = budget_s / len(set(widths))
    rng = np.random.default_rng(0)
    for f in sorted(set(widths)):
        # contiguous row sample with ~target nnz*f work (bounded temporaries)
        target = int(min(3e8 / (8 * f), nnz_total))
        r0 = 0
        r1 = int(np.searchsorted(a_hat.row_ptr, target))
        r1 = max(1, min(r1, a_hat.n_rows))
        lo, hi = a_hat.row_ptr[r0], a_hat.row_ptr[r1]
        sub = O.Csr(r1 - r0, a_hat.n_cols, a_hat.row_ptr[r0:r1 + 1] - lo,
                    a_hat.col_idx[lo:hi], a_hat.values[lo:hi])
        h = rng.standard_normal((a_hat.n_cols, f))
        work, t_used, reps = 0, 0.0, 0
        while t_used < per_width or reps == 0:
            t = time.perf_counter()
            O.local_spmm(sub, h)
            t_used += time.perf_counter() - t
            work += sub.nnz * f
            reps += 1
            if reps >= 50:
                break
        rates[f] = work / t_used
    ms = sum(nnz_total * f / rates[f] for f in widths) * 1e3
    sample = (f"oracle-port local_spmm (np.add.at, sparse.py:222) on leading-row samples "
              f"(~{int(3e8 / 8):,} nnz*f elements each) at widths {sorted(set(widths))}; "
              f"full epoch = sum over {len(widths)} phases of nnz*f/rate (estimate)")
    return ms, {f: r for f, r in rates.items()}, sample


def host_info():
    """The CPU the reference arm ran on (nproc, model, RAM)."""
    info = {"nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    info["cpu"] = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemTotal"):
                    info["ram_gb"] = round(int(line.split()[1]) / 2**20, 1)
                    break
    except OSError:
        pass
    return info


REF_DIR = os.path.join(ROOT, "baseline", "_ref")

# scaled-down samples for the reference arm (same average degree
# and widths as the full graph, nnz small enough that one epoch of the
# unchanged reference takes a few seconds on the box's cores)
REF_SAMPLES = {
    "reddit": dict(n_full=232_965, nnz_full=114_848_856, alpha=0.6, cap=21_657, n=4096),
    "products": dict(n_full=2_449_029, nnz_full=123_718_280, alpha=0.55, cap=17_481,
                     n=65_536),
    "papers": dict(n_full=111_059_956, nnz_full=3_230_000_000, alpha=0.7, cap=30_000,
                   n=131_072),
}


def import_reference():
    """The unmodified reference package installed in baseline/_ref
    (`pip install --no-deps --target baseline/_ref <copy of /root/reference/pkg>`),
    or None when it is absent."""
    if not os.path.isdir(os.path.join(REF_DIR, "distgcn")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import distgcn
    if not os.path.abspath(distgcn.__file__).startswith(os.path.abspath(REF_DIR)):
        raise SystemExit(f"distgcn imported from {distgcn.__file__}, not baseline/_ref")
    return distgcn


def ref_epoch_times(D, a_hat, x, y, cfg_kw, p, epochs):
    """Wall time of each epoch of the unchanged reference `distgcn.train`
    (gcn.py:230-302) at p simulated ranks.  Observation only: the per-epoch
    `Comm.ledger_mark` collective (gcn.py:285) is wrapped to timestamp its
    completion on rank 0 -- the moment every rank has finished the epoch.
    Returns (per-epoch seconds, TrainResult)."""
    stamps = []
    orig = D.runtime.Comm.ledger_mark

    def timed_mark(self, label):
        orig(self, label)
        if self.rank == 0:
            stamps.append(time.perf_counter())

    cfg = D.TrainConfig(epochs=epochs, **cfg_kw)
    D.runtime.Comm.ledger_mark = timed_mark
    try:
        t0 = time.perf_counter()
        res = D.train(a_hat, x, y, np.ones(a_hat.n_rows, bool), cfg, p=p)
    finally:
        D.runtime.Comm.ledger_mark = orig
    ts = [t0] + stamps
    return [b - a for a, b in zip(ts[:-1], ts[1:])], res


def reference_measure(args, wl, warmup, steps):
    """Time the unchanged reference (see run_reference).  Returns a dict:
    value (full-workload ms per epoch), ms (measured per-step ms), kind,
    sample, cores, timed (per-epoch seconds), extra."""
    D = import_reference()
    if D is None:
        return None
    from paper_2504_04673_b200 import graphgen
    cores = os.cpu_count() or 1
    cfg_kw = dict(layers=wl["layers"], hidden=wl["hidden"], lr=0.01, seed=1,
                  variant=args.variant)
    if args.workload == "rmat14":
        p = args.gpus * args.ranks_per_gpu
        n, u, v = graphgen.rmat_edges(14, 16, 0)
        a = D.gcn_normalize(_ref_csr(D, graphgen.symmetric_unit(n, u, v)))
        x, y, _ = make_inputs(wl, n)
        ep, res = ref_epoch_times(D, a, x, y, cfg_kw, p, warmup + steps)
        timed = ep[warmup:]
        ms = statistics.median(timed) * 1e3
        return dict(value=ms, ms=ms, kind="measured (full workload)", cores=p, timed=timed,
                    sample=(f"full config 1: unchanged distgcn.train (baseline/_ref), "
                            f"R-MAT-14, {a.nnz:,} nnz, p={p} simulated ranks (threads), "
                            f"{args.variant}"),
                    extra={"ref_p": p, "nnz": int(a.nnz),
                           "loss_first_last": [res.losses[0], res.losses[-1]]})
    sp = REF_SAMPLES[args.workload]
    p = min(cores, 16)
    deg = sp["nnz_full"] / sp["n_full"]
    if getattr(args, "ref_full", False):
        # the full-size graph through the unchanged reference: minutes per
        # epoch, so only on request (validates the sample-based estimate);
        # epoch 0 carries the reference's own setup and is dropped
        a = _ref_csr(D, make_graph(args.workload))
        x, y, _ = make_inputs(wl, a.n_rows)
        log(f"[bench] reference, full graph: n={a.n_rows} nnz={a.nnz:,}, p={p} threads")
        ep, _ = ref_epoch_times(D, a, x, y, cfg_kw, p, 1 + max(1, steps))
        timed = ep[1:]
        ms = statistics.median(timed) * 1e3
        return dict(value=ms, ms=ms, kind="measured (full workload)", cores=p, timed=timed,
                    sample=(f"full {args.workload}-shaped graph: unchanged distgcn.train "
                            f"(baseline/_ref), {a.nnz:,} nnz, p={p} simulated ranks = {p} "
                            f"threads, {args.variant}; epoch 0 (with the reference's setup) "
                            f"dropped"),
                    extra={"ref_p": p, "nnz": int(a.nnz),
                           "setup_plus_first_epoch_s": round(ep[0], 1)})

    def sample_graph(ns):
        g = graphgen.chung_lu_host(ns, int(ns * deg / 2), alpha=sp["alpha"],
                                   max_weight=sp["cap"] * ns / sp["n_full"], seed=0)
        return D.gcn_normalize(_ref_csr(D, g))

    a = sample_graph(sp["n"])
    x, y, _ = make_inputs(wl, a.n_rows)
    log(f"[bench] reference sample: n={a.n_rows} nnz={a.nnz:,}, p={p} threads")
    ep, _ = ref_epoch_times(D, a, x, y, cfg_kw, p, warmup + steps)
    timed = ep[warmup:]
    sample_ms = statistics.median(timed) * 1e3
    full_nnz = sp["nnz_full"] + sp["n_full"]          # + self-loops (gcn_normalize)
    scale = full_nnz / a.nnz
    # linearity check: a half-size sample, 3 epochs (first discarded)
    a2 = sample_graph(sp["n"] // 2)
    x2, y2, _ = make_inputs(wl, a2.n_rows)
    ep2, _ = ref_epoch_times(D, a2, x2, y2, cfg_kw, p, 3)
    half_ms = statistics.median(ep2[1:]) * 1e3
    return dict(
        value=sample_ms * scale, ms=sample_ms, cores=p, timed=timed,
        kind="estimate (measured sample epoch x full nnz / sample nnz)",
        sample=(f"unchanged distgcn.train (baseline/_ref) on a scaled-down "
                f"{args.workload}-shaped Chung-Lu graph: n={a.n_rows:,}, nnz={a.nnz:,} "
                f"(avg degree {a.nnz / a.n_rows:.0f}, same widths {wl['f_in']}/"
                f"{wl['hidden']}/{wl['classes']}), p={p} simulated ranks = {p} threads, "
                f"{args.variant}; value = median sample epoch x {scale:,.1f} "
                f"(full nnz {full_nnz:,} / sample nnz)"),
        extra={"ref_p": p, "sample_nnz": int(a.nnz), "sample_epoch_ms": round(sample_ms, 1),
               "scale_to_full": round(scale, 3),
               "linearity": {"half_sample_nnz": int(a2.nnz),
                             "half_sample_epoch_ms": round(half_ms, 1),
                             "ms_per_mnnz_sample": round(sample_ms / a.nnz * 1e6, 2),
                             "ms_per_mnnz_half_sample": round(half_ms / a2.nnz * 1e6, 2)}})


def cpu_baseline_entry(args, wl, a_hat=None, nnz_total=None):
    """`cpu_baseline` of our arm: the unchanged reference (baseline/_ref) on
    a bounded sample (1 warm-up + 3 timed epochs), else the oracle port's
    np.add.at rate (kind "port")."""
    m = reference_measure(args, wl, 1, 3)
    if m is not None:
        return {"value": round(m["value"], 1), "unit": "ms", "cores": m["cores"],
                "kind": "reference", "value_kind": m["kind"], "sample": m["sample"],
                "host": host_info(), **m["extra"]}
    if a_hat is None:
        return None
    cms, rates, sample = cpu_reference_epoch_ms(a_hat, wl, budget_s=args.ref_budget,
                                                nnz_total=nnz_total)
    return {"value": round(cms, 1), "unit": "ms", "cores": 1, "kind": "port",
            "sample": sample, "host": host_info()}


def run_reference(args, wl):
    """--impl reference: the reference's own CPU implementation, unchanged,
    from baseline/_ref, on the box's host cores.  Rank 0 only.

    * rmat14 (config 1): the full workload -- `distgcn.train` at the
      config's p=4 ranks -- timed directly; `value` is measured.
    * reddit / products / papers (configs 2, 3, 5): the reference cannot run
      them at full size (np.add.at temporaries of nnz*f*8 bytes: ~554 GB for
      Reddit) nor within minutes, so every step is one epoch of the unchanged
      `train` on a scaled-down graph of the same shape (same generator law,
      average degree and layer widths), with p = the host's core count so
      every core is busy (the reference's ranks are threads; np.add.at
      releases the GIL).  `ms_per_step` is that measured sample epoch;
      `value` scales it to the full graph by nnz (the epoch is np.add.at
      work, linear in nnz*f at fixed widths; a second, half-size sample is
      timed to show the linearity) and is labelled an estimate."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    t_all = time.time()
    m = reference_measure(args, wl, args.warmup, args.steps)
    # a CPU-only arm: the GPU idles, so its SM clocks say nothing about this run
    clocks = {"note": "CPU-only arm (the reference is NumPy on the host cores); GPU clocks "
                      "not applicable", "host": host_info()}
    if m is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          "baseline/_ref (the reference package) is not installed"}))
        return 0
    line = {
        "metric": "gcn_epoch_ms", "value": round(m["value"], 3), "unit": "ms",
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(m["ms"], 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": bench_config(args, wl),
        "value_kind": m["kind"],
        "cpu_baseline": {"value": round(m["value"], 3), "unit": "ms", "cores": m["cores"],
                         "kind": "reference", "sample": m["sample"], "host": host_info(),
                         **m["extra"]},
        "e2e": {"value": round(m["value"], 3), "unit": "ms", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "epoch_s_each": [round(t, 3) for t in m["timed"]],
        "clocks": clocks,
        "wall_s": round(time.time() - t_all, 1),
    }
    print(json.dumps(line), flush=True)
    return 0


def _has_nvidia_smi():
    import shutil
    return shutil.which("nvidia-smi") is not None


def _ref_csr(D, a):
    """Our CsrMatrix -> the reference's CsrMatrix (same arrays)."""
    return D.CsrMatrix(a.n_rows, a.n_cols, np.asarray(a.row_ptr, np.int64),
                       np.asarray(a.col_idx, np.int64), np.asarray(a.values, np.float64))


def bench_config(args, wl):
    """The `config` dict, identical in both arms (run details go elsewhere)."""
    p = args.gpus * args.ranks_per_gpu
    return {"workload": wl["desc"], "variant": args.variant, "p": p, "c": args.c}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

_U = {}


def spmm_bytes(vp, rank, f):
    """Compulsory bytes of one rank's local SpMM:
    4(m+1) + 8 nnz + 4 f u + 4 f m, with u = distinct gathered rows."""
    ro = vp.ranks[rank]
    if getattr(ro, "col_ext", None) is None:       # HBM-resident operand: counts kept
        m, nnz, u = ro.n_rows, ro.nnz, ro.u
        return 4 * (m + 1) + 8 * nnz + 4 * f * u + 4 * f * m, u, nnz, m
    m, nnz = ro.n_rows, ro.col_ext.size
    key = (id(vp), rank)
    if key not in _U:
        occ = np.zeros(ro.n_local + ro.halo_rows + 1, dtype=bool)
        occ[ro.col_ext] = True
        _U[key] = int(occ.sum())
    u = _U[key]
    return 4 * (m + 1) + 8 * nnz + 4 * f * u + 4 * f * m, u, nnz, m


def _timed(fn, reps, w):
    """Device time of `reps` calls of fn (CUDA events on the current stream),
    bracketed by host barrier + synchronize; max over processes."""
    import torch
    torch.cuda.synchronize()
    w.host_barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    w.host_barrier()
    ms = e0.elapsed_time(e1) / reps
    return max(w.all_gather_object(ms))


def _papers_sample(g, rows_target_nnz=6_000_000):
    """Leading rows of the first hosted block (columns compacted) as a host
    CsrMatrix: the CPU reference's rate sample for the papers-shaped graph."""
    import paper_2504_04673_b200 as P
    i = min(g.blocks)
    rp, col, val = g.blocks[i]
    k = int(np.searchsorted(rp, rows_target_nnz))
    k = max(1, min(k, len(rp) - 1))
    nz = int(rp[k])
    c = col[:nz].long().cpu().numpy()
    uniq, cc = np.unique(c, return_inverse=True)
    return P.CsrMatrix(k, uniq.size, rp[:k + 1].copy(), cc.astype(np.int64),
                       val[:nz].double().cpu().numpy(), check=False)


def run_papers(args, wl):
    """Config 5 (ogbn-papers100M-shaped): the graph, features and labels are
    generated sharded -- every process builds only its hosted block rows, in
    HBM (sharded.py) -- then the same GcnRun epoch loop is timed."""
    import torch
    import paper_2504_04673_b200 as P
    from paper_2504_04673_b200 import _lib, sharded
    from paper_2504_04673_b200.dist import world
    from paper_2504_04673_b200.engine import pad4
    from paper_2504_04673_b200.gcn import PhaseTimer
    from paper_2504_04673_b200.spmm import device_plan

    w = world().init()
    if w.size != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={w.size}")
    if args.variant not in ("1d-sparse", "1d-oblivious") or args.c != 1:
        raise SystemExit("papers workload: 1D variants only")
    lead = w.proc == 0
    p = args.gpus * args.ranks_per_gpu
    t0 = time.time()
    g = sharded.papers_shaped_sharded(p, seed=0, log=log if lead else None)
    t_gen = time.time() - t0
    log(f"[bench] proc {w.proc}: papers graph nnz={g.nnz_total:,} ({t_gen:.0f}s), "
        f"mem {torch.cuda.memory_allocated() / 2**30:.1f} GiB")
    sample = _papers_sample(g) if lead else None
    x, y = sharded.sharded_inputs(g, wl["f_in"], wl["classes"], seed=1)
    cfg = P.TrainConfig(layers=wl["layers"], hidden=wl["hidden"], lr=0.01, epochs=1, seed=1,
                        variant=args.variant)
    gr = sharded.sharded_gcn_run(g, x, y, wl["f_in"], wl["classes"], cfg)
    t_setup = time.time() - t0
    log(f"[bench] proc {w.proc}: setup {t_setup:.0f}s, "
        f"mem {torch.cuda.memory_allocated() / 2**30:.1f} GiB")
    dims, grid = gr.dims, gr.grid
    gr.run(args.warmup)
    torch.cuda.synchronize()
    w.host_barrier()
    l0 = _lib.launch_count()
    clk = ClockSampler(torch.cuda.current_device())
    holder = {}
    gr.timer = PhaseTimer()                 # per-epoch device times inside the timed region
    ms_epoch = _timed(lambda: holder.__setitem__("run", gr.run(args.steps)), 1, w) / args.steps
    clocks = clk.stop()
    launches = _lib.launch_count() - l0
    torch.cuda.synchronize()
    ev = [e for name, e in gr.timer.events if name == "epoch_start"]
    end = gr.timer.events[-1][1]
    each = [a.elapsed_time(b) for a, b in zip(ev, ev[1:] + [end])]
    slow = {}                               # phases of the slowest timed epoch
    k = int(np.argmax(each))
    marks = gr.timer.events
    starts = [i for i, (nm, _) in enumerate(marks) if nm == "epoch_start"] + [len(marks)]
    seg = marks[starts[k]:starts[k + 1]]
    for (_, e0), (nm, e1) in zip(seg[:-1], seg[1:]):
        slow[nm] = round(slow.get(nm, 0.0) + e0.elapsed_time(e1), 2)
    gr.timer = None
    res = gr.result(holder["run"], args.steps)
    peak_mem = max(w.all_gather_object(torch.cuda.max_memory_allocated()))
    gr.timer = PhaseTimer()
    gr.run(1)
    breakdown = {k: round(v, 3) for k, v in gr.timer.summary().items()}
    gr.timer = None
    # ---- dominant kernel: the 128-wide forward SpMM of layer 1 ---------
    dp = device_plan(gr.dm.fwd, grid, args.variant)
    f0, ld0 = dims[0], pad4(dims[0])
    hs = {r: gr.x[r] for r in dp.local}
    zs = {r: torch.empty_like(hs[r]) for r in dp.local}
    dp.exchange_only(hs, f0, ld0)
    dp.spmm_only(hs, f0, ld0, zs)
    t_spmm = _timed(lambda: dp.spmm_only(hs, f0, ld0, zs), 3, w) / 1e3
    t_xchg = _timed(lambda: dp.exchange_only(hs, f0, ld0), 3, w) / 1e3 if p > 1 else None
    del zs
    tot_b = gather_b = 0
    for r in dp.local:
        b, u, nnz, m = spmm_bytes(dp.vplan, r, f0)
        tot_b += b
        gather_b += 4 * (m + 1) + 8 * nnz + 4 * f0 * nnz + 4 * f0 * m
    peak, peak_src = peaks()
    achieved = tot_b / t_spmm / 1e9
    widths = dims[:-1] + dims[1:]
    spmm_bytes_epoch = sum(w.all_gather_object(
        sum(spmm_bytes(dp.vplan, r, f)[0] for f in widths for r in dp.local)))
    op = gr.dm.fwd
    halo_rows = int(op.counts.sum())
    aware = sum(halo_rows * f for f in widths)
    obl = sum((p - 1) * g.n * f for f in widths)
    exch = None
    if t_xchg is not None:
        snd, rcv = [0] * w.size, [0] * w.size
        for sg in dp.vplan.segments:
            qs, qd = w.proc_of(sg.src, p), w.proc_of(sg.dst, p)
            if qs != qd:
                snd[qs] += sg.count
                rcv[qd] += sg.count
        inter = max(max(snd), max(rcv)) * 4 * f0
        nvl, nvl_src = nvlink_peak()
        exch = {"bound": "nvlink", "achieved": round(inter / t_xchg / 1e9, 1), "peak": nvl,
                "unit": "GB/s", "frac": round(inter / t_xchg / 1e9 / nvl, 4),
                "peak_source": nvl_src, "exchange_ms": round(t_xchg * 1e3, 3),
                "busiest_rank_bytes": int(inter), "f": f0}
    cpu = None
    if lead and not args.no_cpu_baseline:
        cpu = cpu_baseline_entry(args, wl, sample, nnz_total=g.nnz_total)
    if not lead:
        return 0
    line = {
        "metric": "gcn_epoch_ms", "value": round(ms_epoch, 3), "unit": "ms",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_epoch, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args, wl),
        "run_config": {"partition": "block (partition.py:154-161)",
                       "l2": "inputs larger than L2 (H0 = %d MB per GPU)"
                             % (sum(t.numel() for t in gr.x.values()) * 4 // 2**20),
                       "ranks_per_gpu": args.ranks_per_gpu,
                       "halo": "single-buffered (one extra device barrier per phase)"},
        "spmm_hbm_gbs": round(spmm_bytes_epoch / (ms_epoch / 1e3) / 1e9, 1),
        "comm_elements_per_epoch": {"aware": int(aware), "oblivious": int(obl),
                                    "ratio": round(aware / obl, 4) if obl else None},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": ncu_traffic(f"papers_f{f0}_p{p}_c1"),
                     "kernel": "spmm_kernel (layer-1 forward SpMM, f=%d, rank 0)" % f0,
                     "algorithmic_bytes": int(tot_b), "kernel_ms": round(t_spmm * 1e3, 3),
                     "gather_gbs": round(gather_b / t_spmm / 1e9, 1), "peak_source": peak_src},
        "exchange": exch,
        "e2e": None,
        "cpu_baseline": cpu,
        "gpu_launches": int(launches),
        "epoch_breakdown_ms": breakdown,
        "epoch_ms_each_rank0": [round(x, 2) for x in each],
        "epoch_ms_median_rank0": round(float(np.median(each)), 2),
        "slowest_epoch_breakdown_ms": slow,
        "peak_mem_gib": round(peak_mem / 2**30, 1),
        "setup_s": round(t_setup, 1),
        "clocks": clocks,
        "loss": [float(v) for v in res.losses.tolist()],
        "nnz": int(g.nnz_total),
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, wl):
    import torch
    if args.workload == "papers":
        return run_papers(args, wl)
    import paper_2504_04673_b200 as P
    from paper_2504_04673_b200 import _lib
    from paper_2504_04673_b200.dist import world
    from paper_2504_04673_b200.engine import OVERLAP_MIN_F, pad4
    from paper_2504_04673_b200.gcn import GcnRun
    from paper_2504_04673_b200.plan import build_variant_plan
    from paper_2504_04673_b200.spmm import device_plan

    w = world().init()
    if w.size != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={w.size}")
    lead = w.proc == 0
    t_setup = time.time()
    a_hat = make_graph(args.workload, p_in=args.p_in)
    n = a_hat.n_rows
    x, y, mask = make_inputs(wl, n)
    p = args.gpus * args.ranks_per_gpu
    c = args.c
    cfg = P.TrainConfig(layers=wl["layers"], hidden=wl["hidden"], lr=0.01, epochs=1, seed=1,
                        variant=args.variant,
                        reduce_after_transform=args.reduce_after_transform)
    part = None
    part_name = "block"
    k = p // c
    if args.partition == "gvb" and k > 1:
        # the reference's greedy-tv -> GVB (partition.py:257-428), run natively
        t_p = time.time()
        part = P.volume_balanced_refine(a_hat, P.greedy_tv_partition(a_hat, k))
        part_name = f"greedy-tv -> GVB (native, {time.time() - t_p:.0f}s host)"
    elif args.partition == "lpa" or (args.partition == "auto" and args.workload == "products"):
        # graph-derived communities (label propagation on the GPU) packed onto
        # k parts, every part community-ordered (also for k=1: locality)
        from paper_2504_04673_b200.locality import lpa_partition
        t_p = time.time()
        part = lpa_partition(a_hat, k)
        part_name = (f"label-propagation communities -> {k} parts, community-ordered "
                     f"({time.time() - t_p:.1f}s)")
    row_order = {"none": None, "lpa": "lpa"}.get(args.row_order)
    if args.row_order == "auto":
        row_order = "lpa" if (args.workload == "products" and args.partition in ("gvb", "block")) \
            else None
    if row_order:
        part_name += f"; SpMM row order: {row_order} communities of each rank's block"
    gr = GcnRun(a_hat, x, y, mask, cfg, p=p, c=c, partition=part, row_order=row_order)
    log(f"[bench] proc {w.proc}: setup {time.time() - t_setup:.1f}s")
    dims = gr.dims
    grid = gr.grid

    # ---- warm-up + timed epochs (inputs resident in HBM; H of layer 1 is
    #      563 MB > 126 MB L2, so no explicit flush is needed) -------------
    # single process, single rank: the epoch is captured once in a CUDA graph
    # and replayed (same kernels on the same buffers; GcnRun.run_graph)
    use_graph = (args.graph == "on" or (args.graph == "auto" and not w.multi
                                          and not args.reduce_after_transform))
    # several ranks in one process: one host thread drives them in lock step
    lockstep = (p > w.size and not args.reduce_after_transform)
    eager = gr.run_lockstep if lockstep else gr.run
    run_epochs = gr.run_graph if use_graph else eager
    gr.run(args.warmup)
    if use_graph:
        gr.run_graph(1)                                # capture outside the timed region
    torch.cuda.synchronize()
    w.host_barrier()
    l0 = _lib.launch_count()
    clk = ClockSampler(torch.cuda.current_device())
    holder = {}
    torch.cuda.nvtx.range_push("timed_epochs")        # ncu --nvtx-include timed_epochs/
    ms_epoch = _timed(lambda: holder.__setitem__("run", run_epochs(args.steps)), 1, w) / args.steps
    torch.cuda.nvtx.range_pop()
    clocks = clk.stop()
    launches = _lib.launch_count() - l0
    if use_graph:   # replayed launches are not counted by the library: launches per epoch x K
        launches = holder["graph_launches"] = gr._graph_launches * args.steps
    res = gr.result(holder["run"], args.steps)

    # ---- extension: the same training with the transform-first order
    #      (A^T (H W); not the reference's order -- reported separately) ----
    import dataclasses
    tf_ms = None
    if not args.no_transform_first:
        gr_tf = GcnRun.__new__(GcnRun)
        gr_tf.__dict__.update(gr.__dict__)
        gr_tf.cfg = dataclasses.replace(cfg, order="transform-first")
        gr_tf.xent, gr_tf.dense = {}, {}
        gr_tf.run(2)
        tf_ms = _timed(lambda: gr_tf.run(args.steps), 1, w) / args.steps

    # ---- per-phase breakdown of one extra epoch (CUDA events between steps)
    from paper_2504_04673_b200.gcn import PhaseTimer
    gr.timer = PhaseTimer()
    eager(1)
    breakdown = {k: round(v, 3) for k, v in gr.timer.summary().items()}
    gr.timer = None

    # ---- dominant kernel: the f_in-wide forward SpMM of layer 1 ---------
    dp = device_plan(gr.dm.fwd, grid, args.variant)
    f0, ld0 = dims[0], pad4(dims[0])
    hs = {r: gr.x[gr.dm.boundaries[grid.coords(r)[0]][0]:
                 gr.dm.boundaries[grid.coords(r)[0]][1]] for r in dp.local}
    zs = {r: torch.empty_like(hs[r]) for r in dp.local}
    dp.exchange_only(hs, f0, ld0)
    dp.spmm_only(hs, f0, ld0, zs)
    t_spmm = _timed(lambda: dp.spmm_only(hs, f0, ld0, zs), 3, w) / 1e3
    t_xchg = _timed(lambda: dp.exchange_only(hs, f0, ld0), 3, w) / 1e3 if p > 1 else None
    narrow = None
    if p > 1 and dims[1] < OVERLAP_MIN_F:
        # one narrow (single-pass) phase taken apart: the exchange + barrier,
        # each rank's SpMM alone (spread = load imbalance), the whole phase
        f1, ld1 = dims[1], pad4(dims[1])
        h1 = {r: torch.randn(hs[r].shape[0], ld1, device=hs[r].device) for r in dp.local}
        z1 = {r: torch.empty_like(h1[r]) for r in dp.local}
        dp.run(h1, f1, ld1, z1)
        t_x1 = _timed(lambda: dp.exchange_only(h1, f1, ld1), 5, w)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            dp.spmm_only(h1, f1, ld1, z1)
        e1.record()
        torch.cuda.synchronize()
        per_rank = w.all_gather_object(round(e0.elapsed_time(e1) / 5, 3))
        t_ph = _timed(lambda: dp.run(h1, f1, ld1, z1), 5, w)
        narrow = {"f": f1, "exchange_ms": round(t_x1, 3), "spmm_ms_per_process": per_rank,
                  "phase_ms": round(t_ph, 3)}
        del h1, z1
    tot_b, gather_b = 0, 0
    for r in dp.local:
        b, u, nnz, m = spmm_bytes(dp.vplan, r, f0)
        tot_b += b
        gather_b += 4 * (m + 1) + 8 * nnz + 4 * f0 * nnz + 4 * f0 * m
    peak, peak_src = peaks()
    achieved = tot_b / t_spmm / 1e9
    probe = gather_probe(n, ld0) if p == 1 else None

    # ---- all SpMM phases of one epoch (HBM GB/s over the epoch's SpMMs) --
    widths = dims[:-1] + dims[1:]
    spmm_bytes_epoch = sum(spmm_bytes(dp.vplan, r, f)[0] for f in widths for r in dp.local)
    spmm_bytes_epoch = sum(w.all_gather_object(spmm_bytes_epoch))

    # ---- communication volume per epoch: aware vs oblivious (elements) --
    fam = "1d" if args.variant.startswith("1d") else "15d"
    vp_a = build_variant_plan(gr.dm.fwd, grid, f"{fam}-sparse", [])
    vp_o = build_variant_plan(gr.dm.fwd, grid, f"{fam}-oblivious", [])
    aware = sum(vp_a.elements(f) for f in widths)
    obl = sum(vp_o.elements(f) for f in widths)
    exch = None
    if t_xchg is not None:
        # NVLink bytes only (segments between ranks on different GPUs), per
        # GPU; the busiest GPU's max(send, receive) sets the exchange time
        snd, rcv = [0] * w.size, [0] * w.size
        for sg in dp.vplan.segments:
            qs, qd = w.proc_of(sg.src, p), w.proc_of(sg.dst, p)
            if qs != qd:
                snd[qs] += sg.count
                rcv[qd] += sg.count
        inter = max(max(snd), max(rcv)) * 4 * f0
        nvl, nvl_src = nvlink_peak()
        exch = {"bound": "nvlink", "achieved": round(inter / t_xchg / 1e9, 1),
                "peak": nvl, "unit": "GB/s", "frac": round(inter / t_xchg / 1e9 / nvl, 4),
                "peak_source": nvl_src,
                "exchange_ms": round(t_xchg * 1e3, 3), "busiest_rank_bytes": int(inter),
                "f": f0}

    # ---- end to end through the public API with host buffers ------------
    # Every step uploads its inputs (the hosted block rows of the features)
    # from pinned host memory and reads the loss back.  The upload for step
    # k+1 runs on a copy stream into the second of two device buffers while
    # epoch k computes (double-buffered input pipeline); step 0's upload is
    # exposed.  All copies are inside the timed region.
    # one upload per hosted block row (the c replicas of a row group that
    # share this process read the same features)
    blocks = sorted({grid.coords(r)[0] for r in dp.local})
    rows = [gr.dm.boundaries[i] for i in blocks]
    # when the row pitch pads the features noticeably (products: 100 -> 128),
    # the step's inputs cross PCIe unpadded and the device scatters them into
    # the padded pitch; otherwise (Reddit: 602 -> 608) they are uploaded as is
    f_in = dims[0] if gr.x.shape[1] > 1.05 * dims[0] else gr.x.shape[1]
    xh = {i: gr.x[r0:r1, :f_in].contiguous().cpu().pin_memory()
          for i, (r0, r1) in zip(blocks, rows)}
    stage = ({i: torch.empty_like(xh[i], device=gr.x.device) for i in blocks}
             if f_in < gr.x.shape[1] else None)
    xbuf = [gr.x, torch.zeros_like(gr.x)]
    copy_stream = torch.cuda.Stream()
    e2e_steps = max(2, args.steps)               # the same K as the device-timed region
    d2h = [0]
    state = {"k": 0, "ev": None}

    def upload(buf, stream):
        with torch.cuda.stream(stream):
            for i, (r0, r1) in zip(blocks, rows):
                if stage is None:
                    buf[r0:r1].copy_(xh[i], non_blocking=True)
                else:
                    stage[i].copy_(xh[i], non_blocking=True)
                    buf[r0:r1, :f_in].copy_(stage[i])
        ev = torch.cuda.Event()
        ev.record(stream)
        return ev

    def e2e_step():
        k = state["k"]
        cur = xbuf[k % 2]
        if k == 0:
            state["ev"] = upload(cur, torch.cuda.current_stream())
        torch.cuda.current_stream().wait_event(state["ev"])
        if k + 1 < e2e_steps:                     # prefetch the next step's inputs
            copy_stream.wait_stream(torch.cuda.current_stream())
            state["ev"] = upload(xbuf[(k + 1) % 2], copy_stream)
        gr.x = cur
        # eager (the graph's input buffer is fixed, the upload alternates);
        # the step's loss: a device-side sum over every rank, then 16 B to host
        rr = gr.run_lockstep(1, gather=False) if lockstep else gr.run(1, gather=False)
        st = gr.global_stats(rr).cpu()
        d2h[0] += st.numel() * st.element_size()
        state["k"] = k + 1

    e2e_ms = _timed(e2e_step, e2e_steps, w)
    gr.x = xbuf[0]
    h2d = sum(w.all_gather_object(sum(v.numel() * 4 for v in xh.values())))

    # CTA cap of each process's overlapped exchange (engine.OVERLAP_XCHG_K)
    xctas = w.all_gather_object(getattr(dp, "xchg_ctas", 0)) if w.multi else None

    # ---- CPU baseline (rank 0, N=1 only) --------------------------------
    cpu = None
    if lead and args.gpus == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_entry(args, wl, a_hat)
    if not lead:
        return 0
    line = {
        "metric": "gcn_epoch_ms", "value": round(ms_epoch, 3), "unit": "ms",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_epoch, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args, wl),
        "run_config": {"reduce_after_transform": bool(args.reduce_after_transform),
                       "partition": part_name, "rank_map": args.rank_map,
                       "p_in": args.p_in if args.workload == "products" else None,
                       "l2": "inputs larger than L2 (H0 = %d MB)" % (gr.x.numel() * 4 // 2**20),
                       "ranks_per_gpu": args.ranks_per_gpu},
        "spmm_hbm_gbs": round(spmm_bytes_epoch / (ms_epoch / 1e3) / 1e9, 1),
        "comm_elements_per_epoch": {"aware": int(aware), "oblivious": int(obl),
                                    "ratio": round(aware / obl, 4) if obl else None},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": ncu_traffic(f"{args.workload}_f{f0}_p{p}_c{c}"),
                     "kernel": "spmm_kernel (layer-1 forward SpMM, f=%d, rank 0)" % f0,
                     "algorithmic_bytes": int(tot_b), "kernel_ms": round(t_spmm * 1e3, 3),
                     "gather_gbs": round(gather_b / t_spmm / 1e9, 1), "peak_source": peak_src,
                     "gather_probe_gbs": probe,
                     "gather_frac_of_probe": (round(gather_b / t_spmm / 1e9 / probe, 3)
                                              if probe else None)},
        "exchange": exch,
        "e2e": {"value": round(e2e_ms, 3), "unit": "ms", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h[0] // e2e_steps)},
        "cpu_baseline": cpu,
        "gpu_launches": int(launches),
        "cuda_graph": bool(use_graph),
        "overlap_xchg_ctas": xctas,
        "narrow_phase": narrow,
        "host_driver": ("graph" if use_graph else "") + ("+lockstep" if lockstep else "")
                       if (use_graph or lockstep) else "rank threads",
        "epoch_breakdown_ms": breakdown,
        "extension_transform_first": None if tf_ms is None else {
            "epoch_ms": round(tf_ms, 3),
            "note": "TrainConfig(order='transform-first'): A^T (H W) for width-reducing layers; "
                    "same function, forward exchange at the narrow width (volume below the "
                    "reference's aware count); not the reference's order, not the headline"},
        "clocks": clocks,
        "loss": [float(v) for v in res.losses.tolist()],
        "nnz": int(a_hat.nnz),
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="reddit", choices=sorted(WORKLOADS))
    ap.add_argument("--variant", default="1d-sparse")
    ap.add_argument("--ref-budget", type=float, default=15.0)
    ap.add_argument("--ref-full", action="store_true",
                    help="--impl reference: time the unchanged reference on the FULL graph "
                         "(minutes per epoch; validates the sample-based estimate)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ranks-per-gpu", type=int, default=None,
                    help="virtual ranks per GPU (default 1; rmat14: p=4 ranks in total, "
                         "config 1)")
    ap.add_argument("--c", type=int, default=1, help="1.5D replication factor")
    ap.add_argument("--no-transform-first", action="store_true")
    ap.add_argument("--reduce-after-transform", action="store_true",
                    help="extension: 1.5D replica reduction after the transform")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="CUDA-graph-captured epochs (auto: single process, single rank)")
    ap.add_argument("--partition", default="auto", choices=["auto", "block", "lpa", "gvb"],
                    help="auto: block (Reddit) / lpa (products); lpa: label-propagation "
                         "communities packed onto the parts; gvb: the reference's "
                         "greedy-tv -> GVB")
    ap.add_argument("--p-in", type=float, default=0.8,
                    help="products: share of edges inside the planted communities (0.8 = "
                         "configs 3/4; higher values make the sparsity-aware saving visible)")
    ap.add_argument("--rank-map", default="block", choices=["block", "cyclic"],
                    help="virtual rank -> GPU placement (dist.World.rank_map): block keeps "
                         "1.5D replicas on one GPU, cyclic spreads them (NVLink reduction)")
    ap.add_argument("--row-order", default="auto", choices=["auto", "none", "lpa"],
                    help="SpMM processing order of each rank's rows (no effect on results); "
                         "auto: lpa for products under a block / gvb partition")
    args = ap.parse_args()
    os.environ["DG_RANK_MAP"] = args.rank_map
    wl = WORKLOADS[args.workload]
    if args.ranks_per_gpu is None:
        args.ranks_per_gpu = max(1, 4 // args.gpus) if args.workload == "rmat14" else 1
    if args.impl == "reference":
        return run_reference(args, wl)
    return run_ours(args, wl)


if __name__ == "__main__":
    sys.exit(main())
