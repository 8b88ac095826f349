#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (run under gpurun)
O=gpurun_out/${1:-sanitize}
mkdir -p $O
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> $O/sanitizer.txt
  timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_run.py 2>&1 | grep -E "COMPUTE-SANITIZER|sanitize run|SUMMARY|Error|error" | head -20 >> $O/sanitizer.txt
done
for tool in memcheck racecheck; do
  echo "== $tool SV_PAIR=1" >> $O/sanitizer.txt
  SV_PAIR=1 timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_run.py 2>&1 | grep -E "COMPUTE-SANITIZER|sanitize run|SUMMARY|Error|error" | head -20 >> $O/sanitizer.txt
done
cat $O/sanitizer.txt
