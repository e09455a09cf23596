mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_multi.py > gpurun_out/pytest_gpu_c.log 2>&1; echo pytest=$?
tail -6 gpurun_out/pytest_gpu_c.log
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_n1_c.json 2> gpurun_out/bench_n1_c.err; echo bench=$?
timeout 600 python bench.py --workload reddit --steps 100 --warmup 5 > gpurun_out/bench_reddit_n1_c.json 2> gpurun_out/bench_reddit_n1_c.err; echo reddit=$?
timeout 600 python bench.py --workload scale --steps 50 --warmup 5 > gpurun_out/bench_scale_n1_c.json 2> gpurun_out/bench_scale_n1_c.err; echo scale=$?
for s in 0 10 100 -1; do timeout 600 python examples/train_wdl.py --staleness $s --steps 600 >> gpurun_out/train_n1.jsonl 2>> gpurun_out/train_n1.err; done; echo train=$?
cat gpurun_out/train_n1.jsonl
HET_TIMELINE=1 python -c "from paper_2112_07221_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
timeout 600 python tools/timeline.py > gpurun_out/timeline_n1.txt 2>&1; echo timeline=$?
