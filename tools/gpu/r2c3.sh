# round 2, call 3: ncu evidence for cfg2 (on-chip kernel), cfg5 (HBM passes + DRAM traffic)
set -x
python -c "from paper_2404_06314_b200 import build; build.build()" > gpurun_out/r2c3_build.log 2>&1
python tools/profile_one.py --config 2 --rows 1024 > gpurun_out/r2c3_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:vqc_jit_sa -s 1 -c 1 -o gpurun_out/r2_cfg2_sa python tools/profile_one.py --config 2 --rows 1024 > gpurun_out/r2c3_ncu2.log 2>&1
python tools/profile_one.py --config 5 --rows 16 --reps 1 > gpurun_out/r2c3_plain5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:vqc_jit_pa -s 5 -c 1 -o gpurun_out/r2_cfg5_pa python tools/profile_one.py --config 5 --rows 16 --reps 1 > gpurun_out/r2c3_ncu5a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:vqc_jit_pf -s 5 -c 1 -o gpurun_out/r2_cfg5_pf python tools/profile_one.py --config 5 --rows 16 --reps 1 > gpurun_out/r2c3_ncu5f.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_traffic_cfg5.csv python tools/profile_one.py --config 5 --rows 16 --reps 1 > gpurun_out/r2c3_ncu5t.log 2>&1
ls -la gpurun_out/
