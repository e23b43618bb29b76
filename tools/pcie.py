"""PCIe copy throughput probe (tooling): pinned host <-> device, 1..4 streams,
one direction or both at once."""
import time
import torch

N = 1 << 30  # bytes per buffer
h_in = torch.empty(4 * N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(4 * N, dtype=torch.uint8).pin_memory()
d_in = torch.empty(4 * N, dtype=torch.uint8, device="cuda")
d_out = torch.empty(4 * N, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]


def run(ns, h2d=True, d2h=False, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        chunk = 4 * N // ns
        for i in range(ns):
            if h2d:
                with torch.cuda.stream(streams[i]):
                    d_in[i * chunk:(i + 1) * chunk].copy_(h_in[i * chunk:(i + 1) * chunk], non_blocking=True)
            if d2h:
                with torch.cuda.stream(streams[4 + i]):
                    h_out[i * chunk:(i + 1) * chunk].copy_(d_out[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return 4 * N / best / 1e9


for ns in (1, 2, 4):
    print(f"streams={ns} h2d {run(ns):.1f} GB/s  d2h {run(ns, False, True):.1f} GB/s  "
          f"both {run(ns, True, True):.1f} GB/s per direction")
