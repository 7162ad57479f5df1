# compute-sanitizer over every execution path (tools/sanitize_cases.py);
# logs in gpurun_out/sanitize/<tool>_<case>.log
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for c in cluster register tma heavy matrix slabs; do
    timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_cases.py $c > gpurun_out/sanitize/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$?" | tee -a gpurun_out/sanitize/summary.txt
  done
done
