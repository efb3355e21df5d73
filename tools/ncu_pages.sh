#!/bin/bash
# Text pages of an `ncu --set full` capture, one file per kernel:
#   bash tools/ncu_pages.sh gpurun_out/r02_frame.ncu-rep profiles/r02_ncu
set -e
REP=$1; OUT=$2
KS=${3:-k_observation_normals k_hamming k_preselect_orb k_solve_frame}
for k in $KS; do
  ncu -i "$REP" --page details -k regex:"$k" --print-units base > "${OUT}_${k}.txt" 2>/dev/null || true
  ncu -i "$REP" --page raw -k regex:"$k" --csv --metrics \
    gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__pcsamp_warps_issue_stalled_barrier,smsp__average_warp_latency_issue_stalled_barrier \
    > "${OUT}_${k}_raw.csv" 2>/dev/null || true
done
ls -la ${OUT}_*
