#!/bin/bash
# One GPU session: parity suite, bench line, sanitizers (logs -> gpurun_out/)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
if [ -n "$PYTEST_K" ]; then timeout 1500 python -m pytest tests -m gpu -q -k "$PYTEST_K" > gpurun_out/pytest.log 2>&1; else timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; fi
echo "pytest rc=$?" >> gpurun_out/pytest.log
tail -3 gpurun_out/pytest.log
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json
fi
if [ -n "$SANITIZE" ]; then
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_round.py \
      > gpurun_out/sanitize_$tool.log 2>&1
    echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
  done
fi
