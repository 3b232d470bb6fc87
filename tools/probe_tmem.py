import os, sys, torch, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_05832_b200 import _lib
L = _lib.debug_lib()
out = torch.zeros(1, dtype=torch.int64, device="cuda")
for mode in (0, 1):
    for nw in (4, 8, 16):
        for batch in (1, 4):
            res = []
            for iters in (64, 1024):
                L.hla_debug_tmem_rate(nw, iters, mode, batch, ctypes.c_void_p(out.data_ptr()), None)
                torch.cuda.synchronize()
                res.append(int(out.item()))
            per = (res[1] - res[0]) / (1024 - 64)       # cycles per instruction per warp
            bytes_per_clk = nw * 4096 / per
            print("%s warps=%2d batch=%d: %.1f cyc/instr/warp -> %.0f B/clk per SM" % ("ld" if mode == 0 else "st", nw, batch, per, bytes_per_clk))
