cd $GRAFT_REPO_ROOT
for o in rr blocked; do
for c in C4z1.5 C3 C2; do
  CJ_FIND_ORDER=$o timeout 600 python bench.py --config $c --variant phj-gftr --no-extras --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$o $c', round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,2), 'Gt/s frac', round(d['join_roofline']['frac_b_alg'],3), [ (k['kernel'], round(k['ms_per_step'],2)) for k in d['kernels'][:4]])"
done
done
