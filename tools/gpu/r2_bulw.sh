# Bulyan coordinate phase (17 rows at C3) A/B: consumer warps 16 / 24 / 32, ring 200 / 220 KB
cd $GRAFT_REPO_ROOT
cat > /tmp/bul_time.py <<'PY'
import json, os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch
import paper_2010_05888_b200 as gar
import synth
n, f, d = 31, 7, synth.RESNET50_D
X = synth.make_gradients(n, f, d, seed=7, device="cuda")
a = gar.init("bulyan", n, f)
out = torch.empty(d, device="cuda")
idx = torch.arange(17, dtype=torch.int32, device="cuda") * 1
ws = torch.empty(gar.gar_workspace_bytes("bulyan", n, f, d), dtype=torch.uint8, device="cuda")
for _ in range(3):
    gar.gar_combine("bulyan", X, f, 0, idx, out, d=d)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(20):
    gar.gar_combine("bulyan", X, f, 0, idx, out, d=d)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(json.dumps({"variant": os.environ.get("GAR_LIB_VARIANT", "prod"), "bulyan_phase_ms": round(ms, 4),
                  "frac": round((17 * 4 + 4) * d / (ms * 1e-3) / 1e9 / 6533.5, 3)}))
PY
for rep in 1 2; do
for v in prod w16 w32 r220; do
  if [ $v = prod ]; then unset GAR_LIB_VARIANT; else export GAR_LIB_VARIANT=$v; fi
  timeout 300 python /tmp/bul_time.py 2>&1 | tail -1
done; done
