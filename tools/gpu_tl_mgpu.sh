# N=2 graph-step timeline (HET_TIMELINE build, restored after)
HET_TIMELINE=1 python -c "from paper_2112_07221_b200 import build; build.build(force=True)" > gpurun_out/tlm_build.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 tools/timeline_step_mgpu.py > gpurun_out/tlm.txt 2>&1
TL_DENSE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29634 tools/timeline_step_mgpu.py > gpurun_out/tlm_nodense.txt 2>&1
python -c "from paper_2112_07221_b200 import build; build.build(force=True)" >> gpurun_out/tlm_build.log 2>&1
grep rank gpurun_out/tlm.txt | tail -2 | tr '|' '\n'; echo NODENSE; grep rank gpurun_out/tlm_nodense.txt | tail -2
