for sb in 0 3 5 8 12; do echo "== SB=$sb"; CURVKIT_SYMKR_SB=$sb timeout 120 python tools/hess_c1_once.py c1 5 2>&1 | tail -1 | grep -o "'hess_symkr': ([^)]*)"; done
