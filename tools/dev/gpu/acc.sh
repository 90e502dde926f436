set -x
timeout 900 python -m pytest tests/test_acceptance.py tests/test_eigops.py -m gpu -x -q -s 2>&1 | tail -30
CURVKIT_TRACE_LAUNCHES=1 ./oracle/_ref/acceptance_b200 | tail -12
