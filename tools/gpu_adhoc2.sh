cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > /tmp/t.log 2>&1; tail -3 /tmp/t.log
for env in CJ_LOOKBACK=1 CJ_LOOKBACK=0; do echo "== $env"; for c in C2 C4z1.5 C3; do env $env CONFIG=$c timeout 300 python tools/diag.py phj-gftr smj-gftr 2>&1 | grep " 3 wall"; done; done
