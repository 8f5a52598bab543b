mkdir -p gpurun_out
python tools/c2_engines.py 100000 > gpurun_out/c2_engines.log 2>&1
SLOSIM_LANE_LPW=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lane_kernel -c 1 -o gpurun_out/c2_solo -f python tools/c2_one.py 20000 0 > gpurun_out/c2_solo_ncu.log 2>&1
SLOSIM_FORCE_LATENCY_ENGINE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_kernel -c 1 -o gpurun_out/c2_warp -f python tools/c2_one.py 20000 0 > gpurun_out/c2_warp_ncu.log 2>&1
cat gpurun_out/c2_engines.log
