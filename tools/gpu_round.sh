#!/bin/bash
# One GPU-box pass (not part of the product): gpu tests, smoke, bench, ncu launch
# list, one ncu --set full capture of the hot kernels.  Everything lands in gpurun_out/.
# STAGES selects parts: t=tests s=smoke b=bench l=launch lists f=full ncu
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
ST=${STAGES:-tsblf}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt
if [[ $ST == *t* ]]; then
  timeout ${TEST_TIMEOUT:-900} python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
  tail -30 gpurun_out/pytest_gpu.log
fi
if [[ $ST == *s* ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  echo "smoke exit $?" >> gpurun_out/smoke.log
  tail -3 gpurun_out/smoke.log
fi
if [[ $ST == *b* ]]; then
  timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
  tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
  for v in ${EXTRA_VARIANTS:-smj-gftr}; do
    timeout 300 python bench.py --variant $v --no-extras > gpurun_out/bench_$v.json 2>> gpurun_out/bench.err
  done
fi
if [[ $ST == *l* ]]; then
  for v in ${LAUNCH_VARIANTS:-phj-gftr smj-gftr}; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$v.csv python bench.py --steps 2 --warmup 1 --no-extras \
      --variant $v > gpurun_out/launches_$v.log 2>&1
  done
fi
if [[ $ST == *f* ]]; then
  for v in ${FULL_VARIANTS:-phj-gftr smj-gftr}; do
    timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"${NCU_KERNELS:-k_scatter_blocks|k_phj_tma|k_smj_tma|k_block_hist}" -s ${NCU_SKIP:-0} -c ${NCU_COUNT:-5} \
      -o gpurun_out/full_$v -f python bench.py --steps 1 --warmup 0 --no-extras --variant $v \
      > gpurun_out/full_$v.log 2>&1
  done
fi
ls -la gpurun_out
