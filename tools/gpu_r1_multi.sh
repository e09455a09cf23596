# round-1 multi-GPU evidence: run with `gpurun --gpus 4 -- bash tools/gpu_r1_multi.sh`
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
tr() { # torchrun N tag args...
  local N=$1 tag=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29400 + RANDOM % 500)) bench.py --gpus $N "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
  echo "$tag rc=$?"; tail -c 300 gpurun_out/bench_$tag.json; echo
}
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload reddit --steps 100 --warmup 5 > gpurun_out/bench_reddit_n1.json 2> gpurun_out/bench_reddit_n1.err; echo reddit_n1 rc=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --workload scale --steps 100 --warmup 5 > gpurun_out/bench_scale_n1.json 2> gpurun_out/bench_scale_n1.err; echo scale_n1 rc=$?
tr 2 dcn_n2 --steps 100 --warmup 5
tr 4 dcn_n4 --steps 100 --warmup 5
tr 2 reddit_n2 --workload reddit --steps 100 --warmup 5
tr 4 reddit_n4 --workload reddit --steps 100 --warmup 5
tr 2 scale_n2 --workload scale --steps 100 --warmup 5
tr 4 scale_n4 --workload scale --steps 100 --warmup 5
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi.log 2>&1; echo pytest_multi=$?
tail -5 gpurun_out/pytest_multi.log
