# round 2, call 8: device bounds checks (memcheck stand-in); complex64 tile / slot knobs
set -x
python -c "from paper_2404_06314_b200 import build; build.build()" > gpurun_out/r2c8_build.log 2>&1
timeout 1800 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_device_checks.py > gpurun_out/r2c8_checks.log 2>&1
echo "checks rc=$?"
rm -f gpurun_out/r2c8_knobs.log
for spec in "X=0" "VQC_TILE_QUBITS=12 VQC_FWD_TILE=12" "VQC_FWD_TILE=12" "VQC_REG_SLOTS=4 VQC_ADJ_DUAL=1" "VQC_REG_SLOTS=4 VQC_ADJ_DUAL=1 VQC_TILE_QUBITS=12 VQC_FWD_TILE=12" "VQC_JIT_MINB_ADJ=3 VQC_JIT_MINB_FWD=6"; do
  echo "== complex64 $spec cfg4" >> gpurun_out/r2c8_knobs.log
  env VQC_PRECISION=complex64 $spec timeout 400 python tools/time_config.py --config 4 2>&1 | tail -1 | cut -c1-600 >> gpurun_out/r2c8_knobs.log
done
