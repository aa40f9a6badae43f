#!/bin/bash
# Per-kernel counters of one decode of every bench workload (run on the GPU
# box; one ncu pass per workload, the workload's default batch):
#   bash profiles/collect_ncu.sh [workloads...]   -> gpurun_out/ncu_<workload>.csv
# profiles/traffic.py <round> turns the CSVs (copied to profiles/<round>_ncu/)
# into <round>_traffic.json (bench.py reads the newest for the per-kernel
# issue / DRAM fractions and roofline.traffic).
set -u
WLS=${*:-"cfg1 cfg0 cfg2_4.5 cfg2_3.5 cfg2_2.5 cfg3 cfg4_L8 cfg4_L16 cfg4_L32 fa_i8_4.5 fa_i16_4.5"}
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum
M=$M,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active
M=$M,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum
M=$M,sm__warps_active.avg.pct_of_peak_sustained_active
mkdir -p gpurun_out
for w in $WLS; do
  # the first decode of the process: a CA decode is one launch; FA: the SC
  # pass two launches per list rung (its small-pass launch and its
  # regular one, of which only one decodes)
  timeout 900 ncu --metrics $M --clock-control none -k regex:"decode_kernel|sc_lanes_kernel" -c 14 --csv \
    --log-file gpurun_out/ncu_$w.csv python bench.py --workload $w --steps 1 --warmup 0 --no-cpu --e2e-steps 1 --extra none \
    > gpurun_out/ncu_$w.log 2>&1
  echo "$w exit=$?"
done
