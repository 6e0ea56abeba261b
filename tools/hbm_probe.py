"""Empirical HBM ceilings on this B200 for the roofline discussion: a 2 GiB
device copy (read+write, the MEASURED_PEAKS method) and a 2 GiB pure read
(int64 sum), timed with CUDA events, best of 10."""

import json

import torch


def best(fn, reps=10):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


def main():
    n = 2 << 30
    a = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    a64 = a.view(torch.int64)
    ms_copy = best(lambda: b.copy_(a))
    ms_read = best(lambda: a64.sum())
    print(json.dumps({"copy_GBps": round(2 * n / ms_copy / 1e6, 1),
                      "read_GBps": round(n / ms_read / 1e6, 1), "bytes": n}))


if __name__ == "__main__":
    main()
