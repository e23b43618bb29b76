cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --scaling strong --steps 3 --warmup 1 --no-extras > gpurun_out/strong.json 2> gpurun_out/strong.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --sharded --steps 5 --warmup 2 --no-extras > gpurun_out/sharded.json 2> gpurun_out/sharded.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python - <<'PY'
import json
for f in ("strong", "sharded", "bench"):
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, d["scaling"], round(d["ms_per_step"], 3), round(d["value"] / 1e9, 2), d.get("shuffle", {}).get("exchange_ms_max_over_ranks"), d["join_roofline"]["frac_b_alg"])
    except Exception as e:
        print(f, "ERR", e)
PY
