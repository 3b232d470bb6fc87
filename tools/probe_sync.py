"""Dev probe: tcgen05.commit -> mbarrier and warp <-> warp mbarrier handoff latencies (SM cycles)."""
import os, sys, torch, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_05832_b200 import _lib
L = _lib.debug_lib()
out = torch.zeros(1, dtype=torch.int64, device="cuda")
names = {0: "commit (no MMA) -> mbarrier -> wait", 1: "MMA 128x128x16 + commit -> wait",
         2: "warp<->warp mbarrier ping-pong (1 arrive each way)", 3: "ping-pong, 32 arrivals on the way back"}
for mode in range(4):
    L.hla_debug_sync_latency(mode, 2000, ctypes.c_void_p(out.data_ptr()), None)
    torch.cuda.synchronize()
    print("%-55s %6d cycles per round trip" % (names[mode], int(out.item())))
