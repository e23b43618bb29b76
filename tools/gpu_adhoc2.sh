cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
for c in C4z1.5 C4z1.0; do echo "== $c"; CJ_CTA_TIMES=1 CONFIG=$c timeout 300 python tools/diag.py phj-gftr 2>&1 | grep "cta_times n=268\| 3 wall" | tail -4; done
