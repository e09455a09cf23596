mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_n.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_n.log
for w in wdl reddit; do timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-sweep > gpurun_out/bench_${w}_n1_n.json 2> /dev/null; echo $w=$?
tail -1 gpurun_out/bench_${w}_n1_n.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k:(round(v['ms_per_launch']*1e3,1)) for k,v in d['kernels'].items()})"; done
unset CUDA_VISIBLE_DEVICES
bash tools/gpu_r1_m.sh
