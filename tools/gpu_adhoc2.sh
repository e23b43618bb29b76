cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -k "not star" > /tmp/t.log 2>&1; tail -3 /tmp/t.log
for env in CJ_SPECULATE=1 CJ_SPECULATE=0; do echo "== $env"; for c in C2 C4z1.5 C3; do env $env CONFIG=$c timeout 300 python tools/diag.py phj-gftr phj-gfur 2>&1 | grep " 3 wall"; done; done
