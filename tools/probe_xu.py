"""Dev probe: XU-pipe instruction throughput (per SM, one CTA) for the softmax's exp / pack forms."""
import os, sys, torch, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_05832_b200 import _lib
L = _lib.debug_lib()
out = torch.zeros(1, dtype=torch.int64, device="cuda"); sink = torch.zeros(1, dtype=torch.int32, device="cuda")
names = {0: "ex2.f32", 1: "ex2.bf16x2", 2: "ex2.f16x2", 3: "cvt.bf16x2.f32",
         4: "softmax pair (2 ex2.f32 + cvt)", 5: "softmax pair (ex2.bf16x2, ALU pack)", 6: "softmax pair (ex2.bf16x2, cvt pack)"}
for mode in range(7):
    for threads in (256, 1024):
        r = []
        for iters in (64, 1024):
            L.hla_debug_xu_rate(mode, threads, iters, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(sink.data_ptr()), None)
            torch.cuda.synchronize(); r.append(int(out.item()))
        cyc = (r[1] - r[0]) / (1024 - 64)
        per = 16 if mode < 4 else 8   # instances per iteration (modes 4-6: element pairs)
        print("%-40s threads=%4d: %.2f /clk/SM  (%.1f cyc per warp-instance per SMSP)" %
              (names[mode], threads, threads * per / cyc, cyc / (threads / 128) / per))
