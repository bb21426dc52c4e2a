set -x
python -c "from paper_2404_06314_b200 import build; build.build()" > gpurun_out/r2c10_build.log 2>&1
for spec in "VQC_FOLD_THREAD_TARGETS=1"; do
  env NR=64 $spec timeout 300 python tools/gpu/debug_fold.py > gpurun_out/r2c10_debug3.log 2>&1
done
