# round 2, call 4: ping-pong HBM pass kernels — parity first, then timing
set -x
python -c "from paper_2404_06314_b200 import build; build.build()" > gpurun_out/r2c4_build.log 2>&1
timeout 600 python tools/time_config.py --config 4 --rows 2048 > gpurun_out/r2c4_first.log 2>&1
echo "first rc=$?"
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_module.py tests/test_gpu_complex64.py -k "hbm or golden or 13 or 14 or 15 or 24 or kernel_paths or knobs" > gpurun_out/r2c4_tests.log 2>&1
echo "tests rc=$?"
rm -f gpurun_out/r2c4_knobs.log
for spec in "VQC_PINGPONG=1" "VQC_PINGPONG=0"; do
  for c in 4 5; do
    echo "== $spec cfg$c" >> gpurun_out/r2c4_knobs.log
    env $spec timeout 400 python tools/time_config.py --config $c 2>&1 | tail -1 | cut -c1-700 >> gpurun_out/r2c4_knobs.log
  done
done
echo "== pingpong complex64 cfg4" >> gpurun_out/r2c4_knobs.log
VQC_PRECISION=complex64 timeout 400 python tools/time_config.py --config 4 2>&1 | tail -1 | cut -c1-700 >> gpurun_out/r2c4_knobs.log
