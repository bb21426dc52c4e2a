# round 2, call 7: compute-sanitizer memcheck (one tool per call)
set -x
python -c "from paper_2404_06314_b200 import build; build.build()" > gpurun_out/r2c7_build.log 2>&1
SAN_ROWS=8 timeout 900 python tools/sanitize_case.py > gpurun_out/r2c7_plain.log 2>&1 && \
SAN_ROWS=8 VQC_JIT_CACHE=0 timeout 2400 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
  python tools/sanitize_case.py > gpurun_out/r2c7_memcheck.log 2>&1
echo "memcheck rc=$?"
