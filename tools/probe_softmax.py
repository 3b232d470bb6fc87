import os, sys, torch, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_05832_b200 import _lib
L = _lib.debug_lib()
out = torch.zeros(1024, dtype=torch.int64, device="cuda"); sink = torch.zeros(1, dtype=torch.int32, device="cuda")
for blocks in (1, 148, 296, 592):
    r = []
    for iters in (8, 72):
        L.hla_debug_softmax_rate(blocks, iters, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(sink.data_ptr()), None)
        torch.cuda.synchronize(); r.append(float(out[:blocks].float().mean().item()))
    cyc = (r[1] - r[0]) / 64
    print("blocks=%3d: %.0f cycles per 128x128 tile per CTA (MUFU bound alone: 1024)" % (blocks, cyc))
print("with TMEM S load / P store:")
for blocks in (1, 148, 296):
    r = []
    for iters in (8, 72):
        L.hla_debug_softmax_tile(blocks, iters, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(sink.data_ptr()), None)
        torch.cuda.synchronize(); r.append(float(out[:blocks].float().mean().item()))
    print("blocks=%3d: %.0f cycles per tile per CTA" % (blocks, (r[1] - r[0]) / 64))
print("with TMEM S load / P store + a warp issuing MMAs back to back:")
for blocks in (148, 296):
    r = []
    for iters in (8, 72):
        L.hla_debug_softmax_tile(blocks, iters | (1 << 20), ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(sink.data_ptr()), None)
        torch.cuda.synchronize(); r.append(float(out[:blocks].float().mean().item()))
    print("blocks=%3d: %.0f cycles per tile per CTA" % (blocks, (r[1] - r[0]) / 64))
