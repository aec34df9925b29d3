# Shared-memory wavefronts / instruction counts of the config-2 frame kernel for every
# snapshot in variants_lib/ (run on the GPU box): bash tools/ncu_ab.sh [profile_frame args]
M=smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for lib in variants_lib/libwoit_*.so; do
  echo "== $lib"
  WOIT_LIB=$lib ncu --metrics $M --clock-control none -k regex:frame_kernel -c 1 --csv python tools/profile_frame.py --iters 1 "$@" 2>/dev/null | grep -v "^==" | awk -F'","' 'NR>1{print $(NF-2), $NF}' | tr -d '"'
done
