for m in 1 2; do HET_PDL=$m timeout 300 python bench.py --steps 200 --warmup 5 --no-sweep --no-cpu-baseline > gpurun_out/pdl$m.json 2>/dev/null; python -c "
import json; l=json.loads(open('gpurun_out/pdl$m.json').read().strip().splitlines()[-1]); print('pdl $m', l['ms_per_step']*1e3, l['ms_per_step_stream_launch']*1e3)"; done
bash tools/gpu_tl.sh > /dev/null; tail -4 gpurun_out/tl_graph.txt | head -1 | tr '|' '\n'
