# NVRTC option sweep on the final pass kernels (cfg4 / cfg5), one option per run
bash tools/exp_knobs.sh "X=0" "VQC_JIT_OPTS=--restrict" "VQC_JIT_OPTS=--extra-device-vectorization" \
  "VQC_JIT_OPTS=--ptxas-options=--opt-level=4" "VQC_JIT_OPTS=-DVQC_NOOP_REPEAT" > /dev/null
mkdir -p gpurun_out/r02; cp gpurun_out/exp.log gpurun_out/r02/knobs_c13_nvrtc_opts.log
cat gpurun_out/r02/knobs_c13_nvrtc_opts.log | cut -c1-200
