"""Summarise an .ncu-rep (run here): SOL, pipes, stalls, occupancy, DRAM bytes."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sass__inst_executed_local_loads",
        "smsp__inst_executed.sum", "smsp__sass_inst_executed_op_shared_ld.sum"]
stall_prefix = "smsp__average_warps_issue_stalled_"
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    print("=" * 80)
    for k in want:
        if k in d:
            print(f"{k:70s} {d[k]} {u.get(k, '')}")
    stalls = [(k[len(stall_prefix):], float(d[k])) for k in hdr
              if k.startswith(stall_prefix) and k.endswith("_per_issue_active.ratio") and d[k] not in ("", "n/a")]
    stalls.sort(key=lambda x: -x[1])
    print("stalls per issued instr:", ", ".join(f"{k.replace('_per_issue_active.ratio','')}={v:.2f}" for k, v in stalls[:10]))
