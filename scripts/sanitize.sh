#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2009_10863_b200.build import build; build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -c 'SANITIZE RUN OK' gpurun_out/sanitize_$tool.log) $(grep -E 'ERROR SUMMARY|Error' gpurun_out/sanitize_$tool.log | tail -1)"
done
