"""Dev probe: tile-load throughput per SM for TMA box / gather4 / cp.async / bulk copies."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_05832_b200 import _lib
lib = _lib.debug_lib()
rows, heads = 16 * 4096, 8
src = torch.randn(rows, heads, 64, device="cuda").to(torch.bfloat16)
ctas = torch.cuda.get_device_properties(0).multi_processor_count
cyc = torch.zeros(4 * ctas, dtype=torch.int64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
def M(kind, W=1, nb=0, two=0, pf=0): return kind | (W << 4) | (nb << 8) | (two << 9) | (pf << 10)
cases = [("tma3d W1 pf", M(0, 1, 0, 0, 1), 4, 1), ("tma3d W1 pf 2cta", M(0, 1, 0, 0, 1), 4, 2),
         ("g4 W1 pf", M(1, 1, 0, 0, 1), 4, 1), ("g4 W4 pf", M(1, 4, 0, 0, 1), 4, 1), ("g4 W8 nb pf", M(1, 8, 1, 0, 1), 4, 1), ("tma3d W2", M(0, 2), 4, 1), ("tma3d W2 2maps", M(0, 2, 0, 1), 4, 1), ("tma3d W4 2maps", M(0, 4, 0, 1), 4, 1),
         ("g4 W2", M(1, 2), 4, 1), ("g4 W2 2maps", M(1, 2, 0, 1), 4, 1), ("g4 W4 2maps", M(1, 4, 0, 1), 4, 1),
         ("tma3d W1 st8", M(0), 8, 1), ("tma3d W2 st8 2maps", M(0, 2, 0, 1), 8, 1), ("tma3d W1", M(0), 4, 1), ("tma3d W1 2cta", M(0), 4, 2), ("tma3d W4", M(0, 4), 4, 1),
         ("tma3d W4 nb", M(0, 4, 1), 4, 1), ("g4 W1", M(1), 4, 1), ("g4 W1 2cta", M(1), 4, 2),
         ("g4 W4", M(1, 4), 4, 1), ("g4 W4 nb", M(1, 4, 1), 4, 1), ("g4 W8 nb", M(1, 8, 1), 4, 1),
         ("g4 W8 nb 2cta", M(1, 8, 1), 4, 2), ("g4 W4 nb 8st", M(1, 4, 1), 8, 1),
         ("cp.async", M(2, 4), 4, 1), ("cp.async nb", M(2, 4, 1), 4, 1), ("bulk", M(3), 4, 1)]
for name, mode, stages, per_sm in cases:
    if True:
        tiles = 64
        def run():
            rc = lib.hla_debug_load_rate(src.data_ptr(), rows, heads, mode, stages, ctas * per_sm, tiles, cyc.data_ptr(), None)
            assert rc == 0, rc
        run(); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); run(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = min(ts)
        byts = ctas * per_sm * tiles * 16384
        c = cyc[:ctas * per_sm].float().mean().item() / per_sm
        print("%-16s st %d  %.1f us  %.0f GB/s  %.1f B/clk/SM" % (name, stages, ms * 1e3, byts / ms / 1e6, tiles * 16384 / c))
