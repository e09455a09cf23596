mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 tools/next_sweeps.py comm > gpurun_out/next3_comm_n2.jsonl 2> gpurun_out/next3_comm_n2.err; echo comm=$?
cat gpurun_out/next3_comm_n2.jsonl | cut -c1-300
