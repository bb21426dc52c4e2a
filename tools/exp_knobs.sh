# GPU knob sweep for cfg4/cfg5 (time_config.py); usage: bash tools/exp_knobs.sh "ENV=.. ENV=.." ...
mkdir -p gpurun_out; rm -f gpurun_out/exp.log
for spec in "$@"; do
  for c in 4 5; do
    echo "== $spec cfg$c" >> gpurun_out/exp.log
    env $spec timeout 300 python tools/time_config.py --config $c 2>&1 | cut -c1-330 >> gpurun_out/exp.log
  done
done
cat gpurun_out/exp.log
