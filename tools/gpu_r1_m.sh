mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/pytest_multi_m.log 2>&1; echo pytest_multi=$?
tail -3 gpurun_out/pytest_multi_m.log
for w in reddit dcn; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29400 + RANDOM % 500)) bench.py --gpus 2 --steps 100 --warmup 5 --workload $w > gpurun_out/bench_${w}_n2_m.json 2> /dev/null; echo $w=$?
tail -1 gpurun_out/bench_${w}_n2_m.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k:(round(v['ms_per_launch']*1e3,1)) for k,v in d['kernels'].items()})"; done
