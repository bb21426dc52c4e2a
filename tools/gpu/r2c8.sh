# round 2, call 8: compute-sanitizer racecheck (one tool per call)
set -x
python -c "from paper_2404_06314_b200 import build; build.build()" > gpurun_out/r2c8_build.log 2>&1
SAN_ROWS=4 timeout 900 python tools/sanitize_case.py > gpurun_out/r2c8_plain.log 2>&1 && \
SAN_ROWS=4 VQC_JIT_CACHE=0 timeout 3000 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python tools/sanitize_case.py > gpurun_out/r2c8_racecheck.log 2>&1
echo "racecheck rc=$?"
