cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err; tail -c 600 gpurun_out/ref_arm.json
for v in phj-gftr smj-gftr; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$v.csv python bench.py --steps 2 --warmup 1 --no-extras --variant $v > gpurun_out/launches_$v.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scatter_v2 -s 3 -c 1 -o /tmp/scat -f python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
python tools/ncu_sum.py /tmp/scat.ncu-rep > gpurun_out/ncu_scatter.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_phj_tma -s 0 -c 1 -o /tmp/fill -f python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
python tools/ncu_sum.py /tmp/fill.ncu-rep > gpurun_out/ncu_fill.txt 2>&1
cat gpurun_out/ncu_scatter.txt gpurun_out/ncu_fill.txt
ls -la gpurun_out
