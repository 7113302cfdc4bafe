"""Measure this box's NVLink: 1 GiB peer copies (copy engines,
cudaMemcpyPeerAsync via torch), one direction and both directions at once,
and an all-to-all among all visible GPUs (every GPU copies 1/N GiB to every
peer concurrently).  Prints one JSON line (profiles/ keeps the result).

    python scripts/nvlink_probe.py      # needs >= 2 visible GPUs
"""
import json

import torch


def _time(fn, reps=5):
    for d in range(torch.cuda.device_count()):
        torch.cuda.synchronize(d)
    fn()
    for d in range(torch.cuda.device_count()):
        torch.cuda.synchronize(d)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream(0))
    for _ in range(reps):
        fn()
    for d in range(torch.cuda.device_count()):
        torch.cuda.synchronize(d)
    e1.record(torch.cuda.current_stream(0))
    torch.cuda.synchronize(0)
    return e0.elapsed_time(e1) / reps / 1e3


def main():
    n = torch.cuda.device_count()
    if n < 2:
        print(json.dumps({"error": "needs >= 2 GPUs"}))
        return
    nb = 1 << 30
    bufs = [torch.empty(nb // 4, dtype=torch.float32, device=f"cuda:{d}") for d in range(n)]
    dst = [torch.empty(nb // 4, dtype=torch.float32, device=f"cuda:{d}") for d in range(n)]
    streams = [torch.cuda.Stream(device=f"cuda:{d}") for d in range(n)]

    def one_way():
        with torch.cuda.stream(streams[0]):
            dst[1].copy_(bufs[0], non_blocking=True)

    def both_ways():
        with torch.cuda.stream(streams[0]):
            dst[1].copy_(bufs[0], non_blocking=True)
        with torch.cuda.stream(streams[1]):
            dst[0].copy_(bufs[1], non_blocking=True)

    chunk = nb // 4 // n

    def all_to_all():
        for s in range(n):
            with torch.cuda.stream(streams[s]):
                for k in range(1, n):
                    d = (s + k) % n          # rotated: one sender per receiver at a time
                    dst[d][s * chunk:(s + 1) * chunk].copy_(bufs[s][d * chunk:(d + 1) * chunk],
                                                            non_blocking=True)

    t1 = _time(one_way)
    t2 = _time(both_ways)
    t3 = _time(all_to_all)
    a2a_bytes = (n - 1) * chunk * 4          # per GPU, each direction
    print(json.dumps({
        "gpus": n,
        "peer_copy_one_way_gbs": round(nb / t1 / 1e9, 1),
        "peer_copy_bidirectional_gbs_per_direction": round(nb / t2 / 1e9, 1),
        "all_to_all_gbs_per_gpu_per_direction": round(a2a_bytes / t3 / 1e9, 1),
        "bytes": nb,
    }), flush=True)


if __name__ == "__main__":
    main()
