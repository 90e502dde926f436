for d in 0 1 2 3 6; do echo "DEV_PAIR=$d"; CURVKIT_DEV_PAIR=$d timeout 600 python tools/dev/eigops_time.py 2>&1 | grep "ldh\|materialize P=25450 k=100 tf32 full=False"; done
