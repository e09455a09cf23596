mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
timeout 1500 python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_multi.py > gpurun_out/pytest_gpu_d.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_gpu_d.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-sweep > gpurun_out/bench_n1_d.json 2> gpurun_out/bench_n1_d.err; echo bench=$?
timeout 900 python tools/next_sweeps.py light > gpurun_out/light_sweep.jsonl 2> gpurun_out/light_sweep.err; echo light=$?
cat gpurun_out/light_sweep.jsonl
unset CUDA_VISIBLE_DEVICES
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/pytest_multi_d.log 2>&1; echo pytest_multi=$?
tail -4 gpurun_out/pytest_multi_d.log
for s in 0 10 100 -1; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) examples/train_wdl.py --staleness $s --steps 600 >> gpurun_out/train_n2.jsonl 2>> gpurun_out/train_n2.err; done; echo train=$?
cat gpurun_out/train_n2.jsonl
