# compute-sanitizer over tools/sanitize_run.py; summaries in gpurun_out/san_*.txt
export SAN_STEPS=${SAN_STEPS:-12}
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool --kernel-name kns=het:: --print-limit 20 \
      python tools/sanitize_run.py > gpurun_out/san_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.txt
done
