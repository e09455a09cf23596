mkdir -p gpurun_out
for c in 8 16 32; do HET_NCCL_CTAS=$c timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700 + c)) bench.py --gpus 2 --steps 100 --warmup 5 > gpurun_out/bench_dcn_n2_ctas$c.json 2> gpurun_out/bench_dcn_n2_ctas$c.err; echo ctas$c=$?; tail -1 gpurun_out/bench_dcn_n2_ctas$c.json | cut -c1-250; done
