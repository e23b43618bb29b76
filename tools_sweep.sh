#!/bin/bash
# knob sweep on the GPU box (not part of the product)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
run() {
  echo "=== $*"
  env "$@" timeout 120 python bench.py --steps 8 --warmup 2 --no-extras 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline())
print('ms', round(d['ms_per_step'],3), 'Gt/s', round(d['value']/1e9,2), ' '.join(f\"{k['kernel']}={k['ms_per_step']:.3f}\" for k in d['kernels'][:7]))"
}
timeout 700 python -m pytest tests -x -q -m gpu -k "not dropin" 2>&1 | tail -3
run X=1
run CJ_SCATTER_CTAS=1 CJ_SCATTER_ITEMS=8
run CJ_SCATTER_STAGES=1
run CJ_SCATTER_ITEMS=2
run CJ_SCATTER_CTAS=1 CJ_SCATTER_ITEMS=4
run CJ_FIND_CTAS=2 CJ_FIND_STAGES=1
run CJ_FIND_CTAS=2 CJ_QCHUNK=2048
run CJ_FIND_STAGES=1
run CJ_QCHUNK=2048
echo "=== smj"; timeout 120 python bench.py --steps 4 --warmup 1 --no-extras --variant smj-gftr 2>&1 | tail -1 | cut -c1-1500
