python -m pytest tests/test_gpu_loopback.py -x -q 2>&1 | tail -2
bash tools/gpu_multi2.sh
