timeout 1500 ncu --set full --import-source on --clock-control none -k regex:kr_kernel -c 2 -o gpurun_out/c4_kr python tools/c4_profile.py > gpurun_out/kr_ncu.log 2>&1; echo "rc=$?"
ls -la gpurun_out/c4_kr.ncu-rep
