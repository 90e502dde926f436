set -x
nproc; lscpu | grep -i "model name\|socket\|numa\|^CPU(s)" | head
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_abi.py tests/test_gpu_sketch_pins.py -m gpu -x -q 2>&1 | tail -3
for t in 16 8 32; do CURVKIT_HOST_TIMING=1 CURVKIT_HOST_THREADS=$t timeout 900 python bench.py --no-extra --no-cpu-baseline --steps 3 --warmup 3 --e2e-steps 3 2>&1 | grep -o '"e2e": {[^}]*}\|\[curvkit\] assemble_opg download [0-9.]* ms' | tail -4; done
CURVKIT_FULL_DOWNLOAD=1 CURVKIT_HOST_TIMING=1 timeout 900 python bench.py --no-extra --no-cpu-baseline --steps 3 --warmup 3 --e2e-steps 3 2>&1 | grep -o '"e2e": {[^}]*}\|\[curvkit\] assemble_opg download [0-9.]* ms' | tail -4
