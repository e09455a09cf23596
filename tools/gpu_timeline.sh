set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "graph_replay" 2>&1 | tail -5 > gpurun_out/t3.log
HET_TIMELINE=1 python -c "from paper_2112_07221_b200 import build; build.build(force=True)" > gpurun_out/tlbuild.log 2>&1
python tools/timeline.py > gpurun_out/tl.txt 2>&1; python tools/timeline.py --graph > gpurun_out/tlg.txt 2>&1
python -c "from paper_2112_07221_b200 import build; build.build(force=True)" >> gpurun_out/tlbuild.log 2>&1
cat gpurun_out/t3.log gpurun_out/tl.txt gpurun_out/tlg.txt
