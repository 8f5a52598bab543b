# compute-sanitizer passes over the engine on small batches (GPU box): memcheck, synccheck, racecheck, initcheck.
mkdir -p gpurun_out
TOOLS=${TOOLS:-memcheck synccheck racecheck initcheck}
for tool in $TOOLS; do
  echo "== $tool"
  n=60; [ $tool = initcheck ] && n=12
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py $n > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run" gpurun_out/sanitize_$tool.log | tail -3
done
