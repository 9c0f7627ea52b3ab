for d in 0 1 2 4 5 6 7; do echo "dbg $d"; HS_TC_DBG=$d timeout 60 python tools/conv_probe.py --cin 64 --cout 64 --H 64 --W 64 | tail -1; done
