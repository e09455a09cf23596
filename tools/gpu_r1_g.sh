mkdir -p gpurun_out
tr() { local tag=$1; shift
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29400 + RANDOM % 500)) bench.py --gpus 2 --steps 100 --warmup 5 "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
  echo "$tag rc=$?"; tail -1 gpurun_out/bench_$tag.json | cut -c 1-240; echo; }
tr dcn_n2_p2pdense
HET_DENSE_NCCL=1 tr dcn_n2_nccldense
HET_NCCL_CTAS=8 tr dcn_n2_p2pdense8
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/pytest_multi_g.log 2>&1; echo pytest_multi=$?
tail -4 gpurun_out/pytest_multi_g.log
