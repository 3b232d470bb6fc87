import os, sys, torch, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_05832_b200 import _lib
L = _lib.debug_lib()
out = torch.zeros(1, dtype=torch.int64, device="cuda")
for N in (64, 128, 256):
    for a_mn, b_mn, a_tm in ((0, 0, 0), (0, 0, 2), (1, 1, 2), (0, 1, 1), (0, 1, 3)):
        res = []
        for iters in (64, 512):
            st = L.hla_debug_mma_rate(N, iters, a_mn, b_mn, a_tm, ctypes.c_void_p(out.data_ptr()), None)
            torch.cuda.synchronize()
            res.append(int(out.item()))
        per = (res[1] - res[0]) / (512 - 64)
        print("N=%3d a_mn=%d b_mn=%d a_tmem=%d : %.1f cycles/MMA  -> %.0f flop/clk (peak 8192)" % (N, a_mn, b_mn, a_tm, per, 2 * 128 * N * 16 / per))
