# round 2, call 6: full GPU suite on the new defaults + bench
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2c6_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=10 > gpurun_out/r2c6_gpu_tests.log 2>&1
echo "tests rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2c6_bench.log 2> gpurun_out/r2c6_bench.err
echo "bench rc=$?"
