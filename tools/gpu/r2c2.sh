# round 2, call 2: complex64 parity, peaks (FFMA), adjoint knob sweep on cfg4
set -x
python -c "from paper_2404_06314_b200 import build; build.build()" > gpurun_out/r2c2_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_peaks tools/probe_peaks.cu && /tmp/probe_peaks > gpurun_out/r2c2_peaks.json 2>&1
timeout 1500 python -m pytest tests/test_gpu_complex64.py -x -q -p no:cacheprovider > gpurun_out/r2c2_c64_tests.log 2>&1
echo "c64 tests rc=$?"
rm -f gpurun_out/r2c2_knobs.log
for spec in "X=0" "VQC_REG_SLOTS=4 VQC_ADJ_DUAL=1 VQC_JIT_MINB_ADJ=3" "VQC_REG_SLOTS=4 VQC_ADJ_DUAL=1 VQC_JIT_MINB_ADJ=2" "VQC_REG_SLOTS=4 VQC_ADJ_DUAL=1 VQC_TILE_QUBITS=12 VQC_JIT_MINB_ADJ=1"; do
  for c in 4; do
    echo "== $spec cfg$c" >> gpurun_out/r2c2_knobs.log
    env $spec timeout 400 python tools/time_config.py --config $c 2>&1 | tail -2 | cut -c1-600 >> gpurun_out/r2c2_knobs.log
  done
done
for c in 3 4 5; do
  echo "== complex64 cfg$c" >> gpurun_out/r2c2_knobs.log
  VQC_PRECISION=complex64 timeout 400 python tools/time_config.py --config $c 2>&1 | tail -2 | cut -c1-600 >> gpurun_out/r2c2_knobs.log
done
