#!/bin/bash
# Round-end GPU checks: compute-sanitizer over every kernel path, the GPU test suite, smoke().
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "== $tool"; timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_run.py 2>&1 | grep -E "sanitize run ok|SUMMARY|Error|error" | head -5
done > gpurun_out/sanitize.txt 2>&1
timeout 1800 python -m pytest tests/ -q -m gpu --durations=15 > gpurun_out/pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/sanitize.txt; tail -2 gpurun_out/smoke.txt
