cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
for a in phj smj; do timeout 300 python tools/big_join.py 2 $a > /tmp/bj.log 2>&1; head -5 /tmp/bj.log; grep -i "error" /tmp/bj.log | head -3; done
