cd $GRAFT_REPO_ROOT
for c in C1 C3 C4z0.5 C4z1.0 C4z1.5; do
 for v in phj-gftr smj-gftr; do
  timeout 600 python bench.py --config $c --variant $v --no-extras --steps 5 --warmup 3 2>gpurun_out/err_$c_$v.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c $v', round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,2), 'Gt/s frac', round(d['join_roofline']['frac_b_alg'],3), 'rows', d['config']['out_rows'], [ (k['kernel'], round(k['ms_per_step'],2)) for k in d['kernels'][:4]])" || tail -3 gpurun_out/err_$c_$v.txt
 done
done
