mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_kernels.py > gpurun_out/san/$tool.txt 2>&1
  echo "exit=$?" >> gpurun_out/san/$tool.txt
done
