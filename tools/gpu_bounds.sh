# 1) the normal build: N=1 parity + loopback; 2) the bounds-checked build (device
# asserts on computed indices; compute-sanitizer is closed on the pool): the
# N=1 parity file + loopback + smoke; the normal build is restored at the end
python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -x -q 2>&1 | tail -3 > gpurun_out/bd_normal.log
HET_DIAG=HET_BOUNDS python -c "from paper_2112_07221_b200 import build; build.build(force=True)" > gpurun_out/bd_build.log 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -x -q 2>&1 | tail -3 > gpurun_out/bd_bounds.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/bd_bounds.log 2>&1
python -c "from paper_2112_07221_b200 import build; build.build(force=True)" >> gpurun_out/bd_build.log 2>&1
echo NORMAL; cat gpurun_out/bd_normal.log; echo BOUNDS; tail -4 gpurun_out/bd_bounds.log
