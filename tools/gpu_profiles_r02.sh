#!/bin/bash
# Round-2 profile capture (OPT-6.7B B=64, hot/cold union): launch lists of one
# polar and one dense step, and `ncu --set full` captures of the SHA kernel,
# the select+union kernel, the gathered UP/DOWN GEMMs, the small-batch GEMV
# (B=1) and the fused router.  Numbers printed under ncu are never bench values.
mkdir -p gpurun_out
NCU="ncu --profile-from-start off --clock-control none"
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_polar.csv \
  python tools/profile_step.py > gpurun_out/prof_polar.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_dense.csv \
  python tools/profile_step.py --mode dense > gpurun_out/prof_dense.log 2>&1
python tools/launch_summary.py gpurun_out/launches_polar.csv gpurun_out/launches_dense.csv > gpurun_out/launch_summary.txt 2>&1
timeout 900 $NCU --set full --import-source on -k regex:sha_mma -s 1 -c 1 -o gpurun_out/r02_full_sha -f \
  python tools/profile_step.py --layers 3 > gpurun_out/ncu_full_sha.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:"topk_union|gather_gemm|head_router" -c 4 -o gpurun_out/r02_full_sel_gg -f \
  python tools/profile_step.py --layers 2 > gpurun_out/ncu_full_sel_gg.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:"gemv_up|topk_union" -c 2 -o gpurun_out/r02_full_gemv_b1 -f \
  python tools/profile_step.py --layers 2 --batch 1 > gpurun_out/ncu_full_gemv.log 2>&1
cat > /tmp/router_one.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2505_14884_b200 import MlpRouter
r = MlpRouter(4096, 16384, seed=3)
x = torch.randn(64, 4096, device="cuda").bfloat16()
hid = torch.empty(64, 1024, dtype=torch.bfloat16, device="cuda")
lg = torch.empty(64, 16384, device="cuda")
for _ in range(3):
    r.fused_into(x, hid, lg)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
r.fused_into(x, hid, lg)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
PY
timeout 600 $NCU --set full -k regex:router_mlp -c 1 -o gpurun_out/r02_full_router -f python /tmp/router_one.py > gpurun_out/ncu_full_router.log 2>&1
ls -la gpurun_out | tail -20
