# Deterministic instruction counts of sim_kernel per variant library (GPU box):
#   bash tools/inst_count.sh lib_a lib_b ...   (names under build/ab/)
for v in "$@"; do
  for p in "1 3" "0 2"; do
    r=$(SLOSIM_LIB=$PWD/build/ab/$v.so timeout 300 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:sim_kernel -s 1 -c 1 --csv python tools/slice_run.py 4096 $p 2>/dev/null | grep -v "^==" | tail -2 | awk -F'","' '{print $(NF-2)"="$NF}' | tr -d '"' | tr '\n' ' ')
    echo "$v pairs [$p]: $r"
  done
done
