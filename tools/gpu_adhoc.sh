cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_shard.py tests/test_gpu_scale.py -x -q > gpurun_out/t_shard.log 2>&1; echo "exit $?" >> gpurun_out/t_shard.log
tail -15 gpurun_out/t_shard.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --sharded --steps 5 --warmup 3 --no-extras > gpurun_out/sharded.json 2> gpurun_out/sharded.err
python -c "
import json; d=json.loads(open('gpurun_out/sharded.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['phases_ms'], d['shuffle']); [print(k) for k in d['kernels'][:6]]"
tail -3 gpurun_out/sharded.err
