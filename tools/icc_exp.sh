M=gpu__time_duration.sum,sm__icc_request_hit_rate.pct,sm__icc_requests.sum,smsp__inst_executed.sum,smsp__pcsamp_warps_issue_stalled_no_instructions,smsp__pcsamp_sample_count,smsp__issue_active.avg.pct_of_peak_sustained_active
for o in "dp,pp,cost" "cost"; do
  ncu --metrics $M --clock-control none -k regex:sim_kernel -s 1 -c 1 --csv python tools/order_one.py "$o" 4096 > gpurun_out/icc_$o.csv 2>/dev/null
  echo "== $o"; grep -v "^==" gpurun_out/icc_$o.csv | awk -F'","' '{print $(NF-2), $NF}'
done
SLOSIM_BLOCKS_PER_SM=1 ncu --metrics $M --clock-control none -k regex:sim_kernel -s 1 -c 1 --csv python tools/order_one.py "dp,pp,cost" 1184 > gpurun_out/icc_1w.csv 2>/dev/null
echo "== 1 block/SM"; grep -v "^==" gpurun_out/icc_1w.csv | awk -F'","' '{print $(NF-2), $NF}'
