cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['ms_per_step'], d['join_roofline'], d['roofline'], d['variants'], d['e2e'], d['cpu_baseline'])"
tail -2 gpurun_out/bench.err
timeout 300 python bench.py --variant smj-gftr --no-extras > gpurun_out/bench_smj.json 2>>gpurun_out/bench.err
for v in phj-gftr smj-gftr; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$v.csv python bench.py --steps 2 --warmup 1 --no-extras --variant $v > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scatter_v2 -s 0 -c 6 -o gpurun_out/full_scatter -f python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_phj_tma -s 0 -c 2 -o gpurun_out/full_find -f python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
ls -la gpurun_out
