"""Time the 2-pass 16-bit partition of C2's S side (key + 2 payloads) through
the primitive API (tooling, not part of the product)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2312_00720_b200 as cj  # noqa: E402

ctx = cj.Context(0)
n = int(os.environ.get("N", 1 << 28))
R, S = cj.gen_pk_fk(ctx, 1 << 27, n, 2, 2, 4, 4, 1.0, 0.0, 42)
for it in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    out = cj.radix_partition_passes(ctx, S.key, list(S.payloads), [(0, 8), (8, 16)])
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"iter {it} partition 2x8 bits of {n} rows x 12 B: {ms:.3f} ms  "
          f"{2 * 2 * 12 * n / ms / 1e6:.0f} GB/s (scatter bytes only)")
    del out
