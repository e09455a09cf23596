#!/bin/bash
# GPU-box jobs of this repo (run under gpurun from the repo root):
#   bash tools/gpu_jobs.sh iter            N=1 parity + loopback, WDL bench line, graph timeline
#   bash tools/gpu_jobs.sh timeline [--reddit]   graph-replay timeline (HET_TIMELINE build, restored after)
#   bash tools/gpu_jobs.sh timeline_mgpu   N=2 per-rank timeline, with and without the dense all-reduce
#   bash tools/gpu_jobs.sh timeline_mgpu_scale   N=2 per-rank timeline at BASELINE configs[4] (D = 4096)
#   bash tools/gpu_jobs.sh multi N         multi-process parity (p2p) + DCN bench lines up to N + Reddit at N
#   bash tools/gpu_jobs.sh wide            wide-row parity (N=1 + loopback) and the scale-shaped bench line
#   bash tools/gpu_jobs.sh wide_sweep A/B ..  scale bench per wide-kernel configuration (ring,F,CH,CTAs/ring,F,CTAs)
#   bash tools/gpu_jobs.sh final           round-end evidence: pytest -m gpu, smoke, bench lines, ncu launch list + full sets
#   bash tools/gpu_jobs.sh bounds          parity + loopback with the bounds-checked build (HET_DIAG=HET_BOUNDS)
#   bash tools/gpu_jobs.sh diag MACRO      timeline of a diagnostic build variant next to the normal one
#   bash tools/gpu_jobs.sh ncu_launches    ncu launch list of 10 WDL steps (after a plain run)
#   bash tools/gpu_jobs.sh ncu_full        ncu --set full of the three N=1 kernels (after a plain run)
set -u
rebuild() { python -c "from paper_2112_07221_b200 import build; build.build(force=True)" >> gpurun_out/build.log 2>&1; }
tl_build() { HET_TIMELINE=1 python -c "from paper_2112_07221_b200 import build; build.build(force=True)" >> gpurun_out/build.log 2>&1; }
summary() {
python - "$1" <<'PY'
import json, sys
l = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "step_us", round(l["ms_per_step"] * 1e3, 2), "value", round(l["value"] / 1e6, 2), "M rows/s",
      "launches/step", l.get("launches_per_step"), "nvlink_900", (l.get("nvlink") or {}).get("frac_of_900_nominal"))
for k, v in l.get("kernels", {}).items():
    print("  ", k, round(v["ms_per_launch"] * 1e3, 2), "us")
PY
}
case "${1:-iter}" in
iter)
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -x -q 2>&1 | tail -3
  timeout 600 python bench.py --steps 100 --warmup 5 --no-sweep --no-cpu-baseline > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err
  summary gpurun_out/it_bench.json
  tl_build; python tools/timeline.py --graph > gpurun_out/it_tlg.txt 2>&1; rebuild
  tail -4 gpurun_out/it_tlg.txt | head -1 | tr '|' '\n' ;;
timeline)
  tl_build; python tools/timeline.py --graph ${2:-} > gpurun_out/tl_graph.txt 2>&1; rebuild
  tail -4 gpurun_out/tl_graph.txt | head -1 | tr '|' '\n' ;;
timeline_mgpu)
  tl_build
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 tools/timeline_step_mgpu.py > gpurun_out/tlm.txt 2>&1
  TL_DENSE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29634 tools/timeline_step_mgpu.py > gpurun_out/tlm_nodense.txt 2>&1
  rebuild; grep rank gpurun_out/tlm.txt | tail -2; echo NODENSE; grep rank gpurun_out/tlm_nodense.txt | tail -2 ;;
timeline_mgpu_scale)
  tl_build
  TL_SCALE=1 TL_DENSE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29635 tools/timeline_step_mgpu.py > gpurun_out/tlm_scale.txt 2>&1
  rebuild; grep rank gpurun_out/tlm_scale.txt | tail -2 ;;
multi)
  N=${2:-2}
  python -m pytest tests/test_gpu_multi.py -x -q -k "1]" 2>&1 | tail -3
  for n in $(seq 2 $N); do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29710 + n)) bench.py --gpus $n --steps 100 --warmup 5 > gpurun_out/bench_dcn_n$n.json 2> gpurun_out/bench_dcn_n$n.err
    summary gpurun_out/bench_dcn_n$n.json
  done
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29725 bench.py --gpus $N --steps 100 --warmup 5 --workload reddit > gpurun_out/bench_reddit_n$N.json 2> gpurun_out/bench_reddit_n$N.err
  summary gpurun_out/bench_reddit_n$N.json
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29726 bench.py --gpus $N --steps 50 --warmup 5 --workload scale > gpurun_out/bench_scale_n$N.json 2> gpurun_out/bench_scale_n$N.err
  summary gpurun_out/bench_scale_n$N.json ;;
wide)
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -x -q -k "scale or wide or heavy or toy_full or graph" 2>&1 | tail -3
  timeout 600 python bench.py --steps 50 --warmup 5 --workload scale --no-sweep --no-cpu-baseline > gpurun_out/wide_bench.json 2> gpurun_out/wide_bench.err
  summary gpurun_out/wide_bench.json
  python tools/prof_step.py --scale --steps 10 > gpurun_out/wide_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/wide_launches.csv python tools/prof_step.py --scale --steps 10 > gpurun_out/wide_ncu.log 2>&1
  echo ncu rc $?
  python tools/launches.py gpurun_out/wide_launches.csv 10 ;;
wide_full)
  python tools/prof_step.py --scale --steps 3 > gpurun_out/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_seg_as|k_mv_as" -c 2 -o gpurun_out/prof_wide python tools/prof_step.py --scale --steps 3 > gpurun_out/ncu.log 2>&1
  tail -2 gpurun_out/ncu.log ;;
wide_sweep)   # wide-row kernel configurations: "seg_cfg/mv_cfg" pairs
  shift
  for pair in "$@"; do
    IFS=, read -r a b c d <<< "${pair%/*}"; IFS=, read -r e f g <<< "${pair#*/}"
    HET_DIAG="AS_SEG_R=$a;AS_SEG_F=$b;AS_SEG_C=$c;AS_SEG_N=$d;AS_MV_R=$e;AS_MV_F=$f;AS_MV_N=$g" python -c "from paper_2112_07221_b200 import build; build.build(force=True)" >> gpurun_out/build.log 2>&1
    timeout 600 python bench.py --steps 50 --warmup 5 --workload scale --no-sweep --no-cpu-baseline > gpurun_out/ws.json 2> gpurun_out/ws.err
    echo "== $pair"; summary gpurun_out/ws.json
  done
  rebuild ;;
final)   # round-end evidence on one GPU (outputs under gpurun_out/final_*)
  python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/final_pytest_gpu.log; cat gpurun_out/final_pytest_gpu.log
  python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
  timeout 900 python bench.py > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err; summary gpurun_out/final_bench_n1.json
  timeout 900 python bench.py --impl reference > gpurun_out/final_reference_n1.json 2> gpurun_out/final_reference_n1.err; tail -c 300 gpurun_out/final_reference_n1.json
  timeout 900 python bench.py --workload scale --no-cpu-baseline > gpurun_out/final_bench_scale_n1.json 2> gpurun_out/final_bench_scale_n1.err; summary gpurun_out/final_bench_scale_n1.json
  python tools/prof_step.py --steps 10 > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/final_launches.csv python tools/prof_step.py --steps 10 > gpurun_out/ncu.log 2>&1
  python tools/launches.py gpurun_out/final_launches.csv 10 > gpurun_out/final_launches_summary.txt; cat gpurun_out/final_launches_summary.txt
  ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_update_fused|k_lookup_fused|k_dd_fused" -c 3 -o gpurun_out/final_prof python tools/prof_step.py --steps 3 > gpurun_out/ncu2.log 2>&1
  python tools/prof_step.py --scale --steps 3 > gpurun_out/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_seg_as|k_mv_as|k_lookup_wide|k_update_fused|k_dd_fused" -c 5 -o gpurun_out/final_prof_scale python tools/prof_step.py --scale --steps 3 > gpurun_out/ncu3.log 2>&1
  ls -la gpurun_out/final_prof*.ncu-rep ;;
xb_sweep)   # extraction blocks of the fused update (HET_XB) at WDL and at configs[4]
  shift
  for x in "$@"; do
    for w in wdl scale; do
      HET_XB=$x timeout 600 python bench.py --steps 100 --warmup 5 --workload $w --no-sweep --no-cpu-baseline > gpurun_out/xb.json 2> gpurun_out/xb.err
      echo "== HET_XB=$x $w"; summary gpurun_out/xb.json | head -1
    done
  done ;;
bounds)
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -x -q 2>&1 | tail -3 > gpurun_out/bd_normal.log
  HET_DIAG=HET_BOUNDS python -c "from paper_2112_07221_b200 import build; build.build(force=True)" >> gpurun_out/build.log 2>&1
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -x -q 2>&1 | tail -3 > gpurun_out/bd_bounds.log
  python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/bd_bounds.log 2>&1
  rebuild; echo NORMAL; cat gpurun_out/bd_normal.log; echo BOUNDS; tail -4 gpurun_out/bd_bounds.log ;;
diag)
  tl_build; python tools/timeline.py --graph > gpurun_out/dg_a.txt 2>&1
  HET_TIMELINE=1 HET_DIAG=$2 python -c "from paper_2112_07221_b200 import build; build.build(force=True)" >> gpurun_out/build.log 2>&1
  python tools/timeline.py --graph > gpurun_out/dg_b.txt 2>&1; rebuild
  echo A; tail -4 gpurun_out/dg_a.txt | head -1 | tr '|' '\n'; echo B; tail -4 gpurun_out/dg_b.txt | head -1 | tr '|' '\n' ;;
ncu_launches)
  python tools/prof_step.py --steps 10 > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/prof_step.py --steps 10 > gpurun_out/ncu.log 2>&1
  python tools/launches.py gpurun_out/launches.csv 10 ;;
ncu_full)
  python tools/prof_step.py --steps 3 > gpurun_out/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_update_fused|k_lookup_fused|k_dd_fused" -c 3 -o gpurun_out/prof python tools/prof_step.py --steps 3 > gpurun_out/ncu.log 2>&1
  tail -2 gpurun_out/ncu.log ;;
*) echo "unknown job $1"; exit 2 ;;
esac
