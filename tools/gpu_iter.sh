# one build -> measure iteration on the GPU box: parity, bench line, graph timeline
python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -x -q 2>&1 | tail -4 > gpurun_out/it_tests.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-sweep --no-cpu-baseline > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err
HET_TIMELINE=1 python -c "from paper_2112_07221_b200 import build; build.build(force=True)" > gpurun_out/it_tlbuild.log 2>&1
python tools/timeline.py --graph > gpurun_out/it_tlg.txt 2>&1
python -c "from paper_2112_07221_b200 import build; build.build(force=True)" >> gpurun_out/it_tlbuild.log 2>&1
cat gpurun_out/it_tests.log
python - <<'PY'
import json
l = json.loads(open("gpurun_out/it_bench.json").read().strip().splitlines()[-1])
print("step_us", l["ms_per_step"] * 1e3, "value", l["value"], "launches/step", l["launches_per_step"], "stream_us", l["ms_per_step_stream_launch"] * 1e3)
print("e2e", l["e2e"])
for k, v in l["kernels"].items(): print(k, round(v["ms_per_launch"] * 1e3, 2), "us", v["achieved_gbs"])
PY
tail -1 gpurun_out/it_tlg.txt | tr '|' '\n'
