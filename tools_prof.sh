#!/bin/bash
# profiling helper run on the GPU box (not part of the product)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
timeout 300 ncu --set full --clock-control none --import-source on \
    -k regex:"k_scatter_blocks|k_block_hist|k_phj_tma|k_scan" -s 0 -c 12 -o gpurun_out/prof_phj \
    python bench.py --steps 1 --warmup 0 --scale-log2 3 --no-extras > gpurun_out/prof_phj.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on \
    -k regex:"k_smj" -s 0 -c 4 -o gpurun_out/prof_smj \
    python bench.py --steps 1 --warmup 0 --scale-log2 3 --no-extras --variant smj-gftr > gpurun_out/prof_smj.log 2>&1
timeout 600 python -m pytest tests -x -q -m gpu -k "not dropin" 2>&1 | tail -5
