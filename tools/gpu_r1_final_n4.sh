# round-1 final multi-GPU evidence on the final code (4xB200)
mkdir -p gpurun_out
tr() { local N=$1 tag=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29400 + RANDOM % 500)) bench.py --gpus $N "$@" > gpurun_out/final_bench_$tag.json 2> gpurun_out/final_bench_$tag.err
  echo "$tag rc=$?"; }
timeout 1800 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/final_pytest_multi.log 2>&1; echo pytest_multi=$?
tail -3 gpurun_out/final_pytest_multi.log
tr 2 dcn_n2 --steps 100 --warmup 5
tr 4 dcn_n4 --steps 100 --warmup 5
tr 2 reddit_n2 --workload reddit --steps 100 --warmup 5
tr 4 reddit_n4 --workload reddit --steps 100 --warmup 5
tr 2 scale_n2 --workload scale --steps 50 --warmup 5
tr 4 scale_n4 --workload scale --steps 50 --warmup 5
