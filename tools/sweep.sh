cd $GRAFT_REPO_ROOT
for c in C3; do
for q in auto 1024 2048; do
if [ $q = auto ]; then unset CJ_QCHUNK; else export CJ_QCHUNK=$q; fi
timeout 600 python bench.py --config $c --variant phj-gftr --no-extras --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c q=$q', round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,2), 'Gt/s frac', round(d['join_roofline']['frac_b_alg'],3), [ (k['kernel'], round(k['ms_per_step'],2)) for k in d['kernels'][:5]])"
done
done
