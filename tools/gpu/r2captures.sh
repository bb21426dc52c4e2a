# ncu evidence on the final code: DRAM traffic of one cfg4 call and --set full captures
mkdir -p gpurun_out/r02
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02/traffic_cfg4.csv python tools/profile_one.py --config 4 --rows 2048 --reps 1 > /dev/null 2>&1
for spec in "4 vqc_jit_pa12 pa12_cfg4 1 1024" "4 vqc_jit_pf3 pf3_cfg4 1 1024" "3 vqc_jit_pa0 pa0_cfg3 1 4096" "3 vqc_jit_pf0 pf0_cfg3 1 4096" "2 vqc_jit_pa0 pa0_cfg2 1 1024" "5 vqc_jit_pa7 pa7_cfg5 1 32"; do
  set -- $spec
  ncu --set full --import-source on --clock-control none -k regex:$2\$ --launch-skip $4 -c 1 -o gpurun_out/r02/ncu_$3 -f python tools/profile_one.py --config $1 --rows $5 --reps 2 > gpurun_out/r02/ncu_$3.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-sweep --no-cpu > gpurun_out/r02/launches_bench.log 2>&1
ls gpurun_out/r02
