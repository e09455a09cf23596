mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench=$?
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv python bench.py --steps 20 --warmup 3 --no-sweep > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:'k_dd_fused|k_lookup_fused|k_update_fused' -c 6 -o gpurun_out/full_n1 python bench.py --steps 20 --warmup 3 --no-sweep > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/pytest_gpu.log
