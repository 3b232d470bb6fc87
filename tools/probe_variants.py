"""Dev probe: fwd / bwd_main kernel times of several builds (HLA_LIB_NAME per process)
on the cfg2 shape for the HWA, WSA and DENSE patterns (plain + fused)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hla_synth, paper_2511_05832_b200 as hla
from paper_2511_05832_b200 import api
B, H, d, g = 16, 8, 64, 64
q, k, v, do = hla_synth.attention_inputs(B, g * g, H, d, device="cuda")
def t_ms(fn, iters=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters
out = []
for kind in ("HWA", "WSA", "DENSE"):
    L = hla.HilbertLocalAttention(kind, g, g, 16, 16, B, H, d, device="cuda", fused=(kind == "HWA"))
    L.forward(q, k, v); L.backward(do)
    if kind == "HWA":
        f = lambda: api.hla_attn_fwd(L.desc, L.mask, q, k, v, 0.0, L.o, L.lse, seq_to_cell=L.s2c)
        b = lambda: api.hla_attn_bwd_main(L.desc, L.mask, q, k, v, do, L.dq, L.dk, L.dv, L.workspace, 0.0, seq_to_cell=L.s2c)
    else:
        f = lambda: api.hla_attn_fwd(L.desc, L.mask, q, k, v, 0.0, L.o, L.lse)
        b = lambda: api.hla_attn_bwd_main(L.desc, L.mask, q, k, v, do, L.dq, L.dk, L.dv, L.workspace, 0.0)
    out.append("%s fwd %.4f bwd %.4f" % (kind, t_ms(f), t_ms(b)))
print(os.environ.get("HLA_LIB_NAME", "libhla.so"), " | ".join(out))
