import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hla_synth, paper_2511_05832_b200 as hla
from paper_2511_05832_b200 import api
B, H, d, g = 16, 8, 64, 64
q, k, v, do = hla_synth.attention_inputs(B, g * g, H, d, device="cuda")
def t_ms(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters
for fused in (True, False):
    L = hla.HilbertLocalAttention("HWA", g, g, 16, 16, B, H, d, device="cuda", fused=fused)
    L.forward(q, k, v); L.backward(do)
    if fused:
        f = lambda: api.hla_attn_fwd(L.desc, L.mask, q, k, v, 0.0, L.o, L.lse, seq_to_cell=L.s2c)
        b = lambda: api.hla_attn_bwd_main(L.desc, L.mask, q, k, v, do, L.dq, L.dk, L.dv, L.workspace, 0.0, seq_to_cell=L.s2c)
    else:
        f = lambda: api.hla_attn_fwd(L.desc, L.mask, L.qs, L.ks, L.vs, 0.0, L.os, L.lse)
        b = lambda: api.hla_attn_bwd_main(L.desc, L.mask, L.qs, L.ks, L.vs, L.dos, L.dqs, L.dks, L.dvs, L.workspace, 0.0)
    print("fused" if fused else "plain", "fwd %.4f ms  bwd_main %.4f ms" % (t_ms(f), t_ms(b)))
# SM clock while the forward runs back to back (~1 s)
import bench
cs = bench.ClockSampler(0)
cs.start()
t0 = __import__("time").time()
while __import__("time").time() - t0 < 1.0:
    for _ in range(50): f()
    torch.cuda.synchronize()
print("clocks during fwd loop:", cs.stop())
