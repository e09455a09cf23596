# timeline of a diagnostic build variant (HET_DIAG=macro[,macro]) next to the normal one
HET_TIMELINE=1 python -c "from paper_2112_07221_b200 import build; build.build(force=True)" > gpurun_out/dg_build.log 2>&1
python tools/timeline.py --graph > gpurun_out/dg_a.txt 2>&1
HET_TIMELINE=1 HET_DIAG=$1 python -c "from paper_2112_07221_b200 import build; build.build(force=True)" >> gpurun_out/dg_build.log 2>&1
python tools/timeline.py --graph > gpurun_out/dg_b.txt 2>&1
python -c "from paper_2112_07221_b200 import build; build.build(force=True)" >> gpurun_out/dg_build.log 2>&1
echo A; tail -4 gpurun_out/dg_a.txt | head -1 | tr '|' '\n' | grep -E "up\.|x\.|plan"; echo B; tail -4 gpurun_out/dg_b.txt | head -1 | tr '|' '\n' | grep -E "up\.|x\.|plan"
