mkdir -p gpurun_out; rm -f gpurun_out/exp.log
run() { echo "== $*" >> gpurun_out/exp.log; env "$@" timeout 300 python tools/time_config.py --config 4 2>&1 | cut -c1-260 >> gpurun_out/exp.log; }
run VQC_X=0
run VQC_REG_SLOTS=3
run VQC_REG_SLOTS=3 VQC_JIT_MINB_ADJ=2 VQC_JIT_MINB_FWD=4
run VQC_JIT_MINB_ADJ=1
run VQC_JIT_MINB_FWD=5 VQC_JIT_MINB_ADJ=3
run VQC_REG_SLOTS=3 VQC_TILE_QUBITS=10 VQC_JIT_MINB_ADJ=3 VQC_JIT_MINB_FWD=6
cat gpurun_out/exp.log
