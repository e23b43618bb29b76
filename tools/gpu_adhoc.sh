cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
rm -f gpurun_out/diag3.log
for c in C4z1.0 C4z1.5; do
  echo "== $c" >> gpurun_out/diag3.log
  CONFIG=$c PERLAUNCH=1 timeout 300 python tools/diag.py phj-gftr smj-gftr >> gpurun_out/diag3.log 2>&1
done
grep -v " [012] wall" gpurun_out/diag3.log
c=C4z1.5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scatter_v2 -s 5 -c 1 -o /tmp/scat_$c -f python bench.py --config $c --steps 1 --warmup 0 --no-extras > gpurun_out/ncu_scat_$c.log 2>&1
python tools/sass_hot.py /tmp/scat_$c.ncu-rep k_scatter_v2 3e5 > gpurun_out/scat_hot_$c.txt 2>&1
python tools/ncu_sum.py /tmp/scat_$c.ncu-rep > gpurun_out/scat_sum_$c.txt 2>&1
cat gpurun_out/scat_sum_$c.txt
