"""e2e leg sweep on the GPU box (tooling): python tools/e2e.py [steps...]"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2312_00720_b200 as cj
ctx = cj.Context(0)
R, S = cj.gen_pk_fk(ctx, 1 << 27, 1 << 28, 2, 2, 4, 4, 1.0, 0.0, 42)
opt = cj.options("phj", "gftr")
for st in [int(x) for x in sys.argv[1:]] or [6, 16]:
    r = bench.e2e_leg(ctx, R, S, opt, steps=st, streams=2)
    print(st, json.dumps(r))
