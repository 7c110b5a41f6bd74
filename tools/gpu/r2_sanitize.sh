# compute-sanitizer over every device path (small sizes), summaries to gpurun_out/
nvidia-smi -L
for tool in racecheck synccheck memcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_paths.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "exit=$?" >> gpurun_out/sanitize_$tool.txt
done
