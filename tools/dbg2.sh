SKG_DEBUG=1 python - <<'PY' > gpurun_out/cfir_dbg2.log 2>&1
import sys, ctypes
sys.path.insert(0, '.')
import paper_2108_03948_b200 as sk
print("lib", sk.LIB_PATH, flush=True)
import numpy as np, torch
from paper_2108_03948_b200 import workloads as W
x = torch.from_numpy(W.cfg3_batch(6, 4096)).cuda()
p = sk.ZoomPlanGPU(4096, 0.4e12, 1.2e12, W.FS, sk.SKG_F64, decimation=8, num_taps=65)
print("plan", flush=True)
try:
    out = p.execute(x)
    print("launched", flush=True)
    torch.cuda.synchronize()
    print("synced", flush=True)
except BaseException as e:
    print("EXC", type(e), e, flush=True)
PY
echo rc=$? >> gpurun_out/cfir_dbg2.log
dmesg 2>/dev/null | tail -5 >> gpurun_out/cfir_dbg2.log
