set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2c1_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2c1_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/r2c1_gpu_tests.log 2>&1
echo "tests rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2c1_bench.log 2> gpurun_out/r2c1_bench.err
echo "bench rc=$?"
