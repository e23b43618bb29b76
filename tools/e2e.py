import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, torch
import paper_2312_00720_b200 as cj
ctx = cj.Context(0)
R, S = cj.gen_pk_fk(ctx, 1 << 27, 1 << 28, 2, 2, 4, 4, 1.0, 0.0, 42)
opt = cj.options("phj", "gftr")
for st in (2, 3):
    r = bench.e2e_leg(ctx, R, S, opt, steps=6, streams=st)
    print(st, json.dumps(r))
