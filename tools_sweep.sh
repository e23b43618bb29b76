cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "radix or sort or partition or run_join or shard" 2>&1 | tail -2
for e in "CJ_RANK=0" "CJ_RANK=1" "CJ_RANK=0 CJ_SCATTER_ITEMS=4" "CJ_SCATTER_V=2"; do
  echo "== $e"
  env $e timeout 60 python tools_part.py 2>&1 | tail -1
done
timeout 120 python tools_diag.py phj-gftr smj-gftr 2>&1 | grep -E " 3 " | cut -c1-220
