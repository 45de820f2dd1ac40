"""Host->device copy rate from pinned memory at the e2e upload's sizes
(config B: 10.2 MB in five arrays): one copy vs five vs two streams."""
import json
import statistics
import time

import torch


def timed(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3


def main():
    sizes = [409604, 1633280, 819200, 816644, 6517792]  # bytes, config B arrays
    total = sum(sizes)
    host = [torch.empty(s, dtype=torch.uint8).pin_memory() for s in sizes]
    dev = [torch.empty(s, dtype=torch.uint8, device="cuda") for s in sizes]
    one_h = torch.empty(total, dtype=torch.uint8).pin_memory()
    one_d = torch.empty(total, dtype=torch.uint8, device="cuda")
    s2 = torch.cuda.Stream()
    big_h = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    big_d = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def five():
        for h, d in zip(host, dev):
            d.copy_(h, non_blocking=True)

    def one():
        one_d.copy_(one_h, non_blocking=True)

    def two_streams():
        dev[4].copy_(host[4], non_blocking=True)
        with torch.cuda.stream(s2):
            for h, d in zip(host[:4], dev[:4]):
                d.copy_(h, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s2)

    def big():
        big_d.copy_(big_h, non_blocking=True)

    out = {}
    for name, fn in [("five_copies", five), ("one_copy", one), ("two_streams", two_streams)]:
        ms = timed(fn)
        out[name] = {"ms": ms, "GB/s": total / ms / 1e6}
    ms = timed(big, 10)
    out["256MiB"] = {"ms": ms, "GB/s": (256 << 20) / ms / 1e6}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
