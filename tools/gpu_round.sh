#!/bin/bash
# One GPU-box pass: gpu tests, smoke, bench, launch list, one ncu --set full capture of the bench's lane_kernel launch.
# usage (on the box): bash tools/gpu_round.sh TAG      (NO_NCU=1 skips the ncu passes, NO_TESTS=1 the tests)
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
lscpu > gpurun_out/${TAG}_lscpu.txt 2>&1
if [ -z "$NO_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/${TAG}_bench_ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:lane_kernel -s 1 -c 1 -o gpurun_out/${TAG}_lane_kernel -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_full.log 2>&1
fi
tail -3 gpurun_out/${TAG}_pytest_gpu.log; tail -2 gpurun_out/${TAG}_smoke.log; tail -2 gpurun_out/${TAG}_bench.log
