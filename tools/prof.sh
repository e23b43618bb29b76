#!/bin/bash
# ncu --set full of selected kernels at C2 (tooling, not part of the product)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
V=${V:-phj-gftr}
for k in ${KERNELS:-k_scatter_v2 k_phj_tma k_block_hist}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-0} -c ${COUNT:-2} \
    -o gpurun_out/prof_${V}_$k -f python bench.py --steps 1 --warmup 0 --no-extras --variant $V \
    > gpurun_out/prof_${V}_$k.log 2>&1
  tail -2 gpurun_out/prof_${V}_$k.log
done
ls -la gpurun_out
