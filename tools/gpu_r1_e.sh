mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 100 --warmup 5 --no-sweep > gpurun_out/bench_n1_e.json 2> gpurun_out/bench_n1_e.err; echo bench1=$?
for s in 0 10 100 -1; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) examples/train_wdl.py --staleness $s --steps 600 >> gpurun_out/train_n2.jsonl 2>> gpurun_out/train_n2.err; done; echo train=$?
cat gpurun_out/train_n2.jsonl
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29731 bench.py --gpus 2 --steps 100 --warmup 5 > gpurun_out/bench_dcn_n2_e.json 2> gpurun_out/bench_dcn_n2_e.err; echo bench=$?
HET_BENCH_NO_DENSE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29732 bench.py --gpus 2 --steps 100 --warmup 5 > gpurun_out/bench_dcn_n2_nodense.json 2> gpurun_out/bench_dcn_n2_nodense.err; echo bench_nd=$?
HET_TIMELINE=1 python -c "from paper_2112_07221_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
TL_DENSE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29733 tools/timeline_step_mgpu.py > gpurun_out/tl_mgpu_dense.txt 2>&1; echo tl=$?
TL_DENSE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29734 tools/timeline_step_mgpu.py > gpurun_out/tl_mgpu_nodense.txt 2>&1; echo tl2=$?
grep rank gpurun_out/tl_mgpu_dense.txt | head -6; grep rank gpurun_out/tl_mgpu_nodense.txt | head -6
