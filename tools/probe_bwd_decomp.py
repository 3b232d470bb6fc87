"""Dev probe: attn_bwd_kernel time of the build named by HLA_LIB_NAME
(decomposition variants `make VARIANT=vN DEFS=-DHLA_BWD_VAR=N`) at cfg2 / cfg3 / cfg4
(fused Hilbert layer, bench shapes) and dense cfg2.  Prints one line per build."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import hla_synth
import paper_2511_05832_b200 as hla
from paper_2511_05832_b200 import api

CASES = [("cfg2", "HWA", 64, 16, 16, 8), ("cfg3", "HSA", 64, 16, 16, 8), ("cfg4", "HNA", 128, 7, 16, 12),
         ("dense2", "DENSE", 64, 1, 16, 8)]
if len(sys.argv) > 1:
    CASES = [c for c in CASES if c[0] in sys.argv[1:]]


def t_ms(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


out = []
for name, kind, g, w, B, H in CASES:
    d = 64
    q, k, v, do = hla_synth.attention_inputs(B, g * g, H, d, device="cuda")
    L = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, device="cuda")
    L.forward(q, k, v)
    L.backward(do)
    s2c = None if os.environ.get("HLA_NO_GATHER") else L.s2c

    def b():
        api.hla_attn_bwd_main(L.desc, L.mask, q, k, v, do, L.dq, L.dk, L.dv, L.workspace, 0.0, seq_to_cell=s2c)
    f = lambda: api.hla_attn_fwd(L.desc, L.mask, q, k, v, 0.0, L.o, L.lse, seq_to_cell=s2c)  # noqa: E731
    out.append("%s bwd %.4f fwd %.4f" % (name, t_ms(b), t_ms(f)))
    del L
print(os.environ.get("HLA_LIB_NAME", "libhla.so"), " | ".join(out), flush=True)
