cd $GRAFT_REPO_ROOT
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --variant smj-gftr --no-extras > gpurun_out/bench_smj.json 2>>gpurun_out/bench.err
for v in phj-gftr smj-gftr; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$v.csv python bench.py --steps 2 --warmup 1 --no-extras --variant $v > /dev/null 2>&1
done
# traffic of every scatter launch of one step (light metric set)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_scatter_v2 -s 0 -c 6 --log-file gpurun_out/scatter_traffic.csv python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scatter_v2 -s 3 -c 1 -o gpurun_out/full_scatter -f python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_phj_tma" -s 0 -c 2 -o gpurun_out/full_find -f python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_smj_tma" -s 0 -c 2 -o gpurun_out/full_smj -f python bench.py --steps 1 --warmup 0 --no-extras --variant smj-gftr > /dev/null 2>&1
ls -la gpurun_out; du -sh gpurun_out
