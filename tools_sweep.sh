cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_star.py tests/test_dropin.py -x -q 2>&1 | tail -5
for v in phj-gftr smj-gftr phj-gfur; do
timeout 600 python bench.py --config STAR3 --variant $v --no-extras --steps 5 --warmup 3 2>gpurun_out/err_star.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('STAR3 $v', round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,2), 'Gt/s frac', round(d['join_roofline']['frac_b_alg'],3), 'rows', d['config']['out_rows'], [ (k['kernel'], round(k['ms_per_step'],2)) for k in d['kernels'][:5]])" || tail -5 gpurun_out/err_star.txt
done
