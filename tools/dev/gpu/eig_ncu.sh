set -x
python tools/dev/eig_mat_once.py || exit 1
ncu --set full --clock-control none --import-source on -k regex:"tc_gemm_pair_kernel|project_kernel|expand_kernel" -o gpurun_out/r02_eigops python tools/dev/eig_mat_once.py > gpurun_out/eig_ncu.log 2>&1
tail -5 gpurun_out/eig_ncu.log
ls -la gpurun_out/
