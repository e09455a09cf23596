# graph-mode timeline only (HET_TIMELINE build, restored after)
HET_TIMELINE=1 python -c "from paper_2112_07221_b200 import build; build.build(force=True)" > gpurun_out/tl_build.log 2>&1
python tools/timeline.py --graph > gpurun_out/tl_graph.txt 2>&1
python -c "from paper_2112_07221_b200 import build; build.build(force=True)" >> gpurun_out/tl_build.log 2>&1
tail -2 gpurun_out/tl_graph.txt | tr '|' '\n'
