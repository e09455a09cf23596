# N=2: parity (p2p only, the default exchange), DCN bench line, graph timeline
python -m pytest tests/test_gpu_multi.py -x -q -k "p2p0 or 1]" 2>&1 | tail -3 > gpurun_out/m_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 100 --warmup 5 > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err
cat gpurun_out/m_tests.log
python - <<'PY'
import json
l = json.loads(open("gpurun_out/m_bench.json").read().strip().splitlines()[-1])
print("step_us", l["ms_per_step"] * 1e3, "value", l["value"], "launches/step", l["launches_per_step"])
print("nvlink", l.get("nvlink"))
for k, v in l["kernels"].items(): print(k, round(v["ms_per_launch"] * 1e3, 2), "us")
PY
bash tools/gpu_tl_mgpu.sh
