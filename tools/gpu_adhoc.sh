cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t_parity.log 2>&1; echo "exit $?" >> gpurun_out/t_parity.log
tail -5 gpurun_out/t_parity.log
for env in "CJ_RANK=1" "CJ_RANK=0" "CJ_SCATTER_WARP=0"; do
  echo "== $env" >> gpurun_out/diag.log
  env $env timeout 300 python tools/diag.py phj-gftr smj-gftr phj-gfur >> gpurun_out/diag.log 2>&1
done
tail -60 gpurun_out/diag.log
timeout 300 python bench.py --config C3 --no-extras --steps 3 --warmup 2 > gpurun_out/c3.json 2>&1
head -c 700 gpurun_out/c3.json
