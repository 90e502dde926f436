# full ncu capture of the fp16 J^T T and J X Khatri-Rao kernels (c4, f16s)
timeout 1500 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:kr_kernel<.bool.1, .bool.1>' -c 1 -o gpurun_out/c4_krf16 python tools/c4_profile.py f16s > gpurun_out/krjt_ncu.log 2>&1; echo "rc=$?"
ls -la gpurun_out/c4_krf16.ncu-rep
