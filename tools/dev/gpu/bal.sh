python - > gpurun_out/bal.txt 2>&1 <<'PY'
import json, sys, torch
sys.path.insert(0, ".")
import bench
print(json.dumps(bench.band_balance(torch, torch.device("cuda", 0), torch.cuda.current_stream()), indent=1))
PY
cat gpurun_out/bal.txt
