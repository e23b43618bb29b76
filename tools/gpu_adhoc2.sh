cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > /tmp/t.log 2>&1; tail -2 /tmp/t.log
for c in C2 C4z1.5 C3; do CONFIG=$c timeout 300 python tools/diag.py phj-gftr 2>&1 | grep " [23] wall"; done
CJ_SPECULATE=0 timeout 300 python tools/diag.py phj-gftr 2>&1 | grep " [23] wall"
