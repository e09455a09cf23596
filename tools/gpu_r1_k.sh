mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "dedup_paths or reddit or toy_full_parity" > gpurun_out/pytest_k.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_k.log
for v in 0 1; do if [ $v = 1 ]; then export HET_DD_CLUSTER=1; fi
timeout 600 python bench.py --workload reddit --steps 100 --warmup 5 --no-sweep > gpurun_out/bench_reddit_k$v.json 2> /dev/null; echo reddit$v=$?
tail -1 gpurun_out/bench_reddit_k$v.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k:(round(v['ms_per_launch']*1e3,1)) for k,v in d['kernels'].items()})"; done
