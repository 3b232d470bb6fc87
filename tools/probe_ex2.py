import os, sys, torch, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_05832_b200 import _lib
L = _lib.debug_lib()
out = torch.zeros(1, dtype=torch.int64, device="cuda"); sink = torch.zeros(1, device="cuda")
for threads in (128, 256, 512, 1024):
    r = []
    for iters in (64, 1024):
        L.hla_debug_ex2_rate(threads, iters, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(sink.data_ptr()), None)
        torch.cuda.synchronize(); r.append(int(out.item()))
    cyc = (r[1] - r[0]) / (1024 - 64)   # cycles per iteration (16 ex2 per thread)
    print("threads=%4d: %.1f ex2/clk/SM" % (threads, threads * 16 / cyc))
