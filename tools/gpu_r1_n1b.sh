mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --ignore=tests/test_gpu_multi.py > gpurun_out/pytest_gpu_b.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu_b.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-sweep > gpurun_out/bench_n1_b.json 2> gpurun_out/bench_n1_b.err; echo bench=$?
timeout 600 python bench.py --workload scale --steps 50 --warmup 5 > gpurun_out/bench_scale_n1_b.json 2> gpurun_out/bench_scale_n1_b.err; echo scale=$?
timeout 600 python bench.py --workload reddit --steps 100 --warmup 5 > gpurun_out/bench_reddit_n1_b.json 2> gpurun_out/bench_reddit_n1_b.err; echo reddit=$?
