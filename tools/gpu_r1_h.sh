mkdir -p gpurun_out
tr() { local tag=$1; shift
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29400 + RANDOM % 500)) bench.py --gpus 2 --steps 100 --warmup 5 --workload dcn > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
  echo "$tag rc=$?"; tail -1 gpurun_out/bench_$tag.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k:(round(v['ms_per_launch']*1e3,1)) for k,v in d['kernels'].items()})"; }
HET_NCCL_CTAS=16 tr h_p2p16
HET_NCCL_CTAS=24 tr h_p2p24
HET_NCCL_CTAS=8 HET_DENSE_NCCL=1 tr h_nccl8
HET_NCCL_CTAS=8 tr h_p2p8
