HET_TIMELINE=1 python -c "from paper_2112_07221_b200 import build; build.build(force=True)" > gpurun_out/tl_build.log 2>&1
python tools/timeline.py --graph --reddit > gpurun_out/tl_rd.txt 2>&1
python -c "from paper_2112_07221_b200 import build; build.build(force=True)" >> gpurun_out/tl_build.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 --no-sweep --no-cpu-baseline --workload reddit > gpurun_out/rd.json 2>/dev/null
python -c "
import json; l=json.loads(open('gpurun_out/rd.json').read().strip().splitlines()[-1]); print('reddit', l['ms_per_step']*1e3, l['value']); [print(k, round(v['ms_per_launch']*1e3,2)) for k,v in l['kernels'].items()]"
