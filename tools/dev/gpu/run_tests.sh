# GPU suite on the box (PYTEST_K selects with -k); log under gpurun_out/
if [ -n "$PYTEST_K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -k "$PYTEST_K" > gpurun_out/r02_gputests.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/r02_gputests.log
tail -15 gpurun_out/r02_gputests.log
