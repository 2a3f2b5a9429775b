#!/bin/bash
# Conformance suite (staged reference unit tests through the rbfdeform alias) and the
# compute-sanitizer tools over tools/sanitize_case.py. Logs in gpurun_out/.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_conformance.py -m gpu -x -q -rf > gpurun_out/conformance.log 2>&1; echo "conformance rc=$?"; tail -3 gpurun_out/conformance.log
for tool in ${TOOLS:-memcheck synccheck racecheck}; do
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
