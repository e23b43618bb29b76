cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo "exit $?" >> gpurun_out/t_all.log
tail -15 gpurun_out/t_all.log
for c in C4z1.5 C2; do
  echo "== $c" >> gpurun_out/diag_pl.log
  CONFIG=$c PERLAUNCH=1 timeout 300 python tools/diag.py phj-gftr >> gpurun_out/diag_pl.log 2>&1
done
grep -v "phj-gftr [012] " gpurun_out/diag_pl.log
