for v in rowt dig2 rowt dig2; do for p in "1 3" "0 2"; do echo -n "$v pairs $p: "; SLOSIM_LIB=$PWD/build/ab/lib_$v.so python tools/slice_run.py 8192 $p; done; done
