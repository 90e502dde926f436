set -x
timeout 600 python tools/dev/eigops_time.py 2>&1 | grep "materialize" | grep -v "f32 full"
CURVKIT_EIG_MAT_LSU=1 timeout 600 python tools/dev/eigops_time.py 2>&1 | grep "materialize" | grep -v "f32 full"
