cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > /tmp/t.log 2>&1; tail -1 /tmp/t.log
for c in C2 C3 C4z1.5; do CONFIG=$c timeout 300 python tools/diag.py phj-gftr phj-gfur 2>&1 | grep " 3 wall"; done
