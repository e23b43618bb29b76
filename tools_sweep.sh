#!/bin/bash
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
timeout 700 python -m pytest tests -x -q -m gpu -k "not dropin" 2>&1 | tail -3
python tools_diag.py phj-gftr smj-gftr 2>&1 | grep -E " [23] "
CJ_SCATTER_ITEMS=4 python tools_diag.py phj-gftr 2>&1 | grep -E " [3] "
CJ_SCATTER_STAGES=1 python tools_diag.py phj-gftr 2>&1 | grep -E " [3] "
