"""Dev probe: time of hla_attn_bwd_preprocess at cfg2 / cfg3 / cfg4 (fused layer shapes)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, hla_synth, paper_2511_05832_b200 as hla
from paper_2511_05832_b200 import api
def t_ms(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters
out=[]
for name, kind, g, w, B, H in [("cfg2","HWA",64,16,16,8),("cfg3","HSA",64,16,16,8),("cfg4","HNA",128,7,16,12)]:
    q, k, v, do = hla_synth.attention_inputs(B, g*g, H, 64, device="cuda")
    L = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, 64, device="cuda")
    L.forward(q, k, v); L.backward(do)
    pre = lambda: api.hla_attn_bwd_preprocess(L.o, do, L.lse, L.workspace, seq_to_cell=L.s2c, mask=L.mask)
    out.append("%s pre %.4f" % (name, t_ms(pre)))
print(" | ".join(out))
