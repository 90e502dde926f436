nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_rate tools/mma_rate.cu && /tmp/mma_rate > gpurun_out/mma_rate.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_pins.py -m gpu -q -x -k "hessian" > gpurun_out/fc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fc_tests.log
for v in "0 x" "3 x" "0 1" "3 1"; do set -- $v
  if [ $2 = 1 ]; then export CURVKIT_HESS_SS192=1; else unset CURVKIT_HESS_SS192; fi
  CURVKIT_DEV_FUSED=$1 timeout 300 python bench.py --config c2 --steps 5 --warmup 2 --no-e2e --no-extra --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('dev $1 ss192 $2', round(k['hess_fused']['ms_per_step'],3), d['clocks']['sm_mhz'])
" >> gpurun_out/fused2.txt
done
tail -n 2 gpurun_out/fc_tests.log; cat gpurun_out/mma_rate.txt gpurun_out/fused2.txt
