"""PCIe duplex microbenchmark: pinned host <-> device copies of 4 GiB, one
direction at a time, both at once (one stream each), and both at once with
each direction split over two or four streams (copy engines)."""
import torch

N = 1 << 29  # int64 elements = 4 GiB
h1 = torch.empty(N, dtype=torch.int64, pin_memory=True)
h2 = torch.empty(N, dtype=torch.int64, pin_memory=True)
d1 = torch.empty(N, dtype=torch.int64, device="cuda")
d2 = torch.empty(N, dtype=torch.int64, device="cuda")


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


streams = [torch.cuda.Stream() for _ in range(8)]


def duplex(k):
    cur = torch.cuda.current_stream()
    part = N // k
    for i in range(k):
        su, sd = streams[i], streams[4 + i]
        su.wait_stream(cur)
        sd.wait_stream(cur)
        with torch.cuda.stream(su):
            d1[i * part:(i + 1) * part].copy_(h1[i * part:(i + 1) * part], non_blocking=True)
        with torch.cuda.stream(sd):
            h2[i * part:(i + 1) * part].copy_(d2[i * part:(i + 1) * part], non_blocking=True)
    for i in range(k):
        cur.wait_stream(streams[i])
        cur.wait_stream(streams[4 + i])


gb = 8 * N / 1e9
t = timed(lambda: d1.copy_(h1, non_blocking=True))
print(f"H2D alone: {gb / (t / 1e3):.1f} GB/s")
t = timed(lambda: h2.copy_(d2, non_blocking=True))
print(f"D2H alone: {gb / (t / 1e3):.1f} GB/s")
for k in (1, 2, 4):
    t = timed(lambda: duplex(k))
    print(f"both at once, {k} stream(s) per direction: {gb / (t / 1e3):.1f} GB/s each way, "
          f"{2 * gb / (t / 1e3):.1f} GB/s total")
