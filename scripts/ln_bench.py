"""LayerNorm fwd/bwd timing at the step's shape (8192 x 768)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_10392_b200 import kernels as K
from gemm_shapes import t_ms
T, d = int(os.environ.get("T", 8192)), int(os.environ.get("D", 768))
x, dy, dres = [torch.randn(T, d, device="cuda").bfloat16() for _ in range(3)]
w, b = torch.randn(d, device="cuda").bfloat16(), torch.randn(d, device="cuda").bfloat16()
y, dx = torch.empty_like(x), torch.empty_like(x)
mean, rstd = torch.empty(T, device="cuda"), torch.empty(T, device="cuda")
dw, db = torch.zeros(d, device="cuda"), torch.zeros(d, device="cuda")
f = t_ms(lambda: K.layernorm_fwd(x, w, b, y, mean, rstd))
bw = t_ms(lambda: K.layernorm_bwd(dy, x, w, mean, rstd, dx, dw, db, dx_accum=dres))
bw0 = t_ms(lambda: K.layernorm_bwd(dy, x, w, mean, rstd, dx, dw, db))
print(json.dumps({"lib": os.environ.get("ZB_LIB_PATH", "default"), "T": T, "d": d,
                  "fwd_us": round(f * 1e3, 1), "fwd_gbs": round(T * d * 4 / f / 1e6),
                  "bwd_resid_us": round(bw * 1e3, 1), "bwd_resid_gbs": round(T * d * 8 / bw / 1e6),
                  "bwd_us": round(bw0 * 1e3, 1), "bwd_gbs": round(T * d * 6 / bw0 / 1e6)}))
