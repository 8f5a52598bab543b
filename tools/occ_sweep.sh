for b in 2 3 4; do echo "== blocks/SM $b"; SLOSIM_BLOCKS_PER_SM=$b python tools/order_one.py "dp,pp,cost" 16384 >/dev/null; SLOSIM_BLOCKS_PER_SM=$b python tools/slice_run.py 16384; done
