cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; head -c 1500 gpurun_out/bench.json; echo; tail -3 gpurun_out/bench.err
timeout 300 python bench.py --variant smj-gftr --no-extras > gpurun_out/bench_smj.json 2>>gpurun_out/bench.err; head -c 600 gpurun_out/bench_smj.json
for v in phj-gftr smj-gftr; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$v.csv python bench.py --steps 2 --warmup 1 --no-extras --variant $v > /dev/null 2>&1
done
KERNELS="k_scatter_v2" SKIP=2 COUNT=2 bash tools_prof.sh > /dev/null 2>&1
