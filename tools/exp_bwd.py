import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hla_synth, paper_2511_05832_b200 as hla
B,H,d,g=16,8,64,64
q,k,v,do = hla_synth.attention_inputs(B,g*g,H,d,device="cuda")
for kind, w in (("HWA",16),("WSA",16)):
    L = hla.HilbertLocalAttention(kind,g,g,w,w,B,H,d,device="cuda")
    L.forward(q,k,v); L.backward(do); torch.cuda.synchronize()
    s2c = L.s2c
    def run():
        hla.api.hla_attn_bwd_main(L.desc, L.mask, q, k, v, do, L.dq, L.dk, L.dv, L.workspace, 0.0, seq_to_cell=s2c)
    for _ in range(3): run()
    torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): run()
    e1.record(); torch.cuda.synchronize()
    print(kind, "flags", os.environ.get("HLA_DBG_BWD","0"), "bwd_main ms %.4f" % (e0.elapsed_time(e1)/10))
