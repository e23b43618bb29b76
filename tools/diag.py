"""Per-step timing diagnosis on the GPU box (not part of the product)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2312_00720_b200 as cj  # noqa: E402
from paper_2312_00720_b200 import _capi as A  # noqa: E402

ctx = cj.Context(0)
L = A.lib()
nr, ns = (1 << 27) >> int(os.environ.get("SCALE", "0")), (1 << 28) >> int(os.environ.get("SCALE", "0"))
# CONFIG=C3|C4z0.5|C4z1.0|C4z1.5|C1 picks a bench.py CONFIGS workload (default C2)
if os.environ.get("CONFIG"):
    import bench
    cfg = bench.CONFIGS[os.environ["CONFIG"]]
    nr, ns = cfg["r"], cfg["s"]
    R, S = bench.gen_config(ctx, cfg, nr, ns)
else:
    R, S = cj.gen_pk_fk(ctx, nr, ns, 2, 2, 4, 4, 1.0, 0.0, 42)
Rc, Sc = cj.coljoin.c_relation(R), cj.coljoin.c_relation(S)
for variant in sys.argv[1:] or ["phj-gftr", "smj-gftr"]:
    opt = cj.options(*variant.split("-"))
    res = A.JoinResult()
    for it in range(4):
        A.check(L.cj_set_kernel_timing(ctx.h, 1), ctx.h, "t")
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(ctx.stream)
        A.check(L.cj_run_join(ctx.h, C.byref(Rc), C.byref(Sc), C.byref(opt), C.byref(res)), ctx.h, "j")
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        names = (C.c_char_p * 4096)(); kms = (C.c_float * 4096)(); kby = (C.c_uint64 * 4096)(); cnt = C.c_int()
        A.check(L.cj_kernel_records(ctx.h, 4096, names, kms, kby, C.byref(cnt)), ctx.h, "r")
        ksum = sum(kms[i] for i in range(cnt.value))
        per = {}
        for i in range(cnt.value):
            per[names[i].decode()] = per.get(names[i].decode(), 0) + kms[i]
        if os.environ.get("PERLAUNCH") and it == 3:
            for i in range(cnt.value):
                print(f"   {names[i].decode():14s} {kms[i]:.3f} ms  {kby[i] / 1e9:.2f} GB")
        print(variant, it, f"wall={1e3*(t1-t0):.2f} event={e0.elapsed_time(e1):.2f} "
              f"phases={res.transform_ns/1e6:.2f}/{res.find_ns/1e6:.2f}/{res.materialize_ns/1e6:.2f} "
              f"kernels={ksum:.2f} n={cnt.value} rows={res.rows}",
              " ".join(f"{k}={v:.2f}" for k, v in sorted(per.items(), key=lambda x: -x[1])[:6]))
        A.check(L.cj_result_free(ctx.h, C.byref(res)), ctx.h, "f")
