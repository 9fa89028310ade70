for sd in 0 1 2; do echo "store_dbg $sd"; TGB_STORE_DBG=$sd TGB_PHASE_CLK=1 timeout 120 python tools/prof_pair.py 2>&1 | tail -2 | head -1; done
