# GPU suite (and optional extra command) on the box; logs under gpurun_out/
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/r02_gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gputests.log
tail -15 gpurun_out/r02_gputests.log
