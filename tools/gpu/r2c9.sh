# round 2, call 9: generalized CNOT folds — parity, then timing; complex64 knob combos
set -x
python -c "from paper_2404_06314_b200 import build; build.build()" > gpurun_out/r2c9_build.log 2>&1
timeout 600 python tools/time_config.py --config 4 --rows 2048 > gpurun_out/r2c9_first.log 2>&1; NR=64 timeout 300 python tools/gpu/debug_fold.py > gpurun_out/r2c9_debug.log 2>&1
echo "first rc=$?"
timeout 2000 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_module.py tests/test_gpu_complex64.py tests/test_gpu_device_checks.py tests/test_basis_groups.py -k "hbm or golden or 13 or 14 or 15 or 16 or 24 or kernel_paths or knobs or full_batch or combined or xy or checks" > gpurun_out/r2c9_tests.log 2>&1
echo "tests rc=$?"
rm -f gpurun_out/r2c9_knobs.log
for spec in "VQC_FOLD_THREAD_TARGETS=1" "VQC_FOLD_THREAD_TARGETS=0"; do
  for c in 4 5; do
    echo "== $spec cfg$c" >> gpurun_out/r2c9_knobs.log
    env $spec timeout 400 python tools/time_config.py --config $c 2>&1 | tail -1 | cut -c1-900 >> gpurun_out/r2c9_knobs.log
  done
done
for spec in "VQC_REG_SLOTS=4 VQC_ADJ_DUAL=1 VQC_TILE_QUBITS=12 VQC_FWD_TILE=12" "VQC_REG_SLOTS=4 VQC_ADJ_DUAL=1 VQC_TILE_QUBITS=12 VQC_FWD_TILE=12 VQC_JIT_MINB_ADJ=2" "VQC_REG_SLOTS=4 VQC_ADJ_DUAL=1 VQC_TILE_QUBITS=12 VQC_FWD_TILE=12 VQC_JIT_MINB_ADJ=3 VQC_JIT_MINB_FWD=3"; do
  for c in 4 5; do
    echo "== complex64 $spec cfg$c" >> gpurun_out/r2c9_knobs.log
    env VQC_PRECISION=complex64 $spec timeout 400 python tools/time_config.py --config $c 2>&1 | tail -1 | cut -c1-600 >> gpurun_out/r2c9_knobs.log
  done
done
