# compute-sanitizer over profiles/scripts/sanitize.py, one log per tool, into
# gpurun_out/sanitize_<tool>.log (copy the summaries into profiles/).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --print-limit 50 \
    python profiles/scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
