"""Dev tool: event timeline of CTA 0 of the bwd (or fwd) kernel from the trace build."""
import ctypes, os, sys
os.environ["HLA_LIB_NAME"] = "libhla_trace.so"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hla_synth, paper_2511_05832_b200 as hla
from paper_2511_05832_b200 import _lib
which = sys.argv[1] if len(sys.argv) > 1 else "bwd"
kind = sys.argv[2] if len(sys.argv) > 2 else "HWA"
B, H, d, g = 16, 8, 64, 64
w = 16
q, k, v, do = hla_synth.attention_inputs(B, g * g, H, d, device="cuda")
L = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, device="cuda", fused=(which != "fwdplain"))
for _ in range(3):
    L.forward(q, k, v); L.backward(do)
torch.cuda.synchronize()
lib = _lib.lib()
lib.hla_debug_trace_dump.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 16384)()
lib.hla_debug_trace_dump(buf, 8192)   # reset
if which == "bwd":
    hla.api.hla_attn_bwd_main(L.desc, L.mask, q, k, v, do, L.dq, L.dk, L.dv, L.workspace, 0.0, seq_to_cell=L.s2c)
elif which == "fwdplain":
    hla.api.hla_attn_fwd(L.desc, L.mask, L.qs, L.ks, L.vs, 0.0, L.os, L.lse)
else:
    hla.api.hla_attn_fwd(L.desc, L.mask, q, k, v, 0.0, L.o, L.lse, seq_to_cell=L.s2c)
torch.cuda.synchronize()
n = lib.hla_debug_trace_dump(buf, 8192)
ev = sorted((buf[2 * i + 1], buf[2 * i]) for i in range(n) if buf[2 * i + 1])
t0 = ev[0][0]
names = {1: "MMA", 2: "CMP", 3: "TMA", 4: "DQW", 5: "TC ", 6: "SM1", 7: "TMQ"}
for t, tag in ev[:400]:
    role, e, gg = tag >> 24, (tag >> 16) & 0xFF, tag & 0xFFFF
    print("%8d  %s ev%d g%d" % (t - t0, names.get(role, role), e, gg))
print("events", n, "span cycles", ev[-1][0] - t0)
