mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "toy_full_parity or generic_fallback or wdl_full or light_lfu or graph_replay or scale_shaped or reddit" > gpurun_out/pytest_i.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_i.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-sweep > gpurun_out/bench_n1_i.json 2> gpurun_out/bench_n1_i.err; echo bench=$?
tail -1 gpurun_out/bench_n1_i.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k:(round(v['ms_per_launch']*1e3,1)) for k,v in d['kernels'].items()})"
HET_TIMELINE=1 python -c "from paper_2112_07221_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
timeout 600 python tools/timeline.py > gpurun_out/timeline_n1_i.txt 2>&1; echo timeline=$?
head -3 gpurun_out/timeline_n1_i.txt
