# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_small.py
out=gpurun_out/sanitizer.txt
echo "compute-sanitizer on tools/sanitize_small.py" > $out
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> $out
  timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_small.py 2>&1 | grep -E "sanitize workload|SUMMARY|Error|error" | head -20 >> $out
done
cat $out
