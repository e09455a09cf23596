mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_l.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_l.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-sweep > gpurun_out/bench_n1_l.json 2> /dev/null; echo bench=$?
tail -1 gpurun_out/bench_n1_l.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k:(round(v['ms_per_launch']*1e3,1)) for k,v in d['kernels'].items()})"
timeout 600 python bench.py --workload reddit --steps 100 --warmup 5 --no-sweep > gpurun_out/bench_reddit_l.json 2> /dev/null; echo reddit=$?
tail -1 gpurun_out/bench_reddit_l.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k:(round(v['ms_per_launch']*1e3,1)) for k,v in d['kernels'].items()})"
