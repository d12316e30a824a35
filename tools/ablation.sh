# NEXT-1 execution-model ablation (Fig. 8 / Fig. 9 / Table 5 on B200): OTPW (registers), OTPW+Shared
# (hybrid smem chunks), OTPTB (block barrier after every stage) on Harris and unsharp; time through bench.py and
# ncu counters (barrier stalls, global loads, occupancy, smem bank conflicts) from one run each.
#   bash tools/ablation.sh <tag>
tag=${1:-abl}
mkdir -p gpurun_out/$tag
M=gpu__time_duration.sum,smsp__warp_issue_stalled_barrier_per_warp_active.pct,smsp__warp_issue_stalled_membar_per_warp_active.pct,smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_wait_per_warp_active.pct,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed.sum,launch__registers_per_thread,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum
for wl in harris unsharp; do
  if [ $wl = harris ]; then B="vec=4,chunks=2,rows=48,prefetch=4"; else B="vec=4,chunks=2,rows=32,prefetch=4"; fi
  V1="OTPW_reg;;$B,warps=4,smem_chunks=0"
  V2="OTPW_shared;;$B,warps=4,smem_chunks=1"
  V3="OTPW_shared2;;$B,warps=4,smem_chunks=2"
  V4="OTPTB;PMG_OTPTB=1;$B,warps=4,smem_chunks=0"
  V5="OTPTB_shared;PMG_OTPTB=1;$B,warps=4,smem_chunks=1"
  for v in "$V1" "$V2" "$V3" "$V4" "$V5"; do
    name=${v%%;*}; rest=${v#*;}; envs=${rest%%;*}; opts=${rest#*;}
    bash tools/bench_variants.sh $tag $wl "$envs;$opts" | sed "s/^/$wl $name /"
    env $envs timeout 600 ncu --metrics $M --clock-control none -k regex:'pmg_g0$' -c 1 --csv --log-file gpurun_out/$tag/ncu_${wl}_$name.csv \
      python tools/run_once.py $wl "$opts" 2 > /dev/null 2>&1
  done
done
python tools/ablation_table.py gpurun_out/$tag > gpurun_out/$tag/table.txt; cat gpurun_out/$tag/table.txt
