cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "partition or sort" > /tmp/t.log 2>&1; tail -1 /tmp/t.log
CJ_SLOTS=warp timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "partition or sort or join" > /tmp/t.log 2>&1; tail -1 /tmp/t.log
for e in CJ_SLOTS=cta CJ_SLOTS=warp; do echo "== $e"; env $e timeout 300 python tools/diag.py phj-gftr smj-gftr 2>&1 | grep " [23] wall"; done
