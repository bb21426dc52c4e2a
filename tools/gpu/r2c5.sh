# round 2, call 5: ping-pong mode 2 (alternating shared-memory phases); small-n knobs
set -x
python -c "from paper_2404_06314_b200 import build; build.build()" > gpurun_out/r2c5_build.log 2>&1
VQC_PINGPONG=2 timeout 600 python tools/time_config.py --config 4 --rows 2048 > gpurun_out/r2c5_first.log 2>&1
echo "first rc=$?"
VQC_PINGPONG=2 timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py -k "golden or 13 or 14 or 15" > gpurun_out/r2c5_tests.log 2>&1
echo "tests rc=$?"
rm -f gpurun_out/r2c5_knobs.log
for spec in "VQC_PINGPONG=2" "VQC_PINGPONG=0"; do
  for c in 4 5; do
    echo "== $spec cfg$c" >> gpurun_out/r2c5_knobs.log
    env $spec timeout 400 python tools/time_config.py --config $c 2>&1 | tail -1 | cut -c1-700 >> gpurun_out/r2c5_knobs.log
  done
done
for spec in "X=0" "VQC_SMEM_CTAS_PER_SM=4" "VQC_SMEM_CTAS_PER_SM=8" "VQC_SMEM_DUAL=1" "VQC_SMEM_DUAL=1 VQC_SMEM_CTAS_PER_SM=4" "VQC_SMEM_DUAL=1 VQC_SMEM_CTAS_PER_SM=8" "VQC_JIT_SMEM_FULL=1"; do
  for c in 2 3; do
    echo "== $spec cfg$c" >> gpurun_out/r2c5_knobs.log
    env $spec timeout 400 python tools/time_config.py --config $c --reps 10 2>&1 | tail -1 | cut -c1-500 >> gpurun_out/r2c5_knobs.log
  done
done
for spec in "X=0" "VQC_JIT=1" "VQC_JIT=1 VQC_SMEM_DUAL=1" "VQC_JIT=1 VQC_SMEM_CTAS_PER_SM=8"; do
  echo "== $spec cfg1" >> gpurun_out/r2c5_knobs.log
  env $spec timeout 400 python tools/time_config.py --config 1 --reps 20 2>&1 | tail -1 | cut -c1-500 >> gpurun_out/r2c5_knobs.log
done
