# round-1 final N=1 evidence on the final code: pytest -m gpu, smoke, bench (driver default + sweep),
# ncu launch list and full-set capture of the hot kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_multi.py > gpurun_out/final_pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/final_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/final_ref_n1.json 2>&1; echo ref=$?
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_n1.csv python bench.py --steps 20 --warmup 3 --no-sweep > gpurun_out/final_ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:'k_dd_fused|k_lookup_fused|k_update_fused' -c 6 -o gpurun_out/final_full_n1 python bench.py --steps 20 --warmup 3 --no-sweep > gpurun_out/final_ncu_full.log 2>&1; echo ncu2=$?
timeout 600 python bench.py --workload reddit --steps 100 --warmup 5 --no-sweep > gpurun_out/final_bench_reddit_n1.json 2> /dev/null; echo reddit=$?
timeout 600 python bench.py --workload scale --steps 50 --warmup 5 --no-sweep > gpurun_out/final_bench_scale_n1.json 2> /dev/null; echo scale=$?
