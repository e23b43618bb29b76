"""Large single-GPU join check (tooling): python tools/big_join.py K ALGO [total_bits]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2312_00720_b200 as cj  # noqa: E402

k, algo = int(sys.argv[1]), sys.argv[2]
tb = int(sys.argv[3]) if len(sys.argv) > 3 else -1
ctx = cj.Context(0)
R, S = cj.gen_pk_fk(ctx, 1 << (27 + k), 1 << (28 + k), 2, 2, 4, 4, 1.0, 0.0, 42)
torch.cuda.synchronize()
print("gen ok", flush=True)
out = cj.run_join(ctx, R, S, algo, "gftr", total_radix_bits=tb)
print(k, algo, tb, out.matches, flush=True)
