cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 300 python tools/diag.py phj-gftr smj-gftr phj-gfur smj-gfur 2>&1 | grep " 3 " | cut -c1-250
