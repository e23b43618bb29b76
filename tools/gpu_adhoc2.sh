cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
for g in 32 24 16 12; do echo "== group $g"; CJ_GROUP_BYTES=$g CONFIG=C3 timeout 300 python tools/diag.py phj-gftr smj-gftr 2>&1 | grep " 3 wall"; done
