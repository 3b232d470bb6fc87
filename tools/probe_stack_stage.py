"""Dev probe (GPU): per-stage fwd / bwd times of the cfg5 HWT-T stack with and without the
global-RPB score_mod, to attribute the stack's backward time (DESIGN 6d).  Not a bench line."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hla_synth  # noqa: E402
import paper_2511_05832_b200 as hla  # noqa: E402

B, d = 128, 32
dev = torch.device("cuda", 0)
for g, H, w in [(56, 3, 7), (28, 6, 7), (14, 12, 7), (8, 24, 8)]:
    q, k, v, do = hla_synth.attention_inputs(B, g * g, H, d, seed=1, device=dev)
    for kind in ("HWA", "HSWA"):
        for rpb in (False, True):
            lay = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, shift=(w * w) // 2 if kind == "HSWA" else 0,
                                            device=dev, rpb=rpb)
            if rpb:
                lay.rpb.copy_(torch.rand(lay.rpb.shape) * 2 - 1)
            times = {}

            def mark(name, ev=[]):
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ev.append((name, e))
                return ev
            for it in range(6):
                ev = mark("start", [])
                lay.step(q, k, v, do, lambda n: mark(n, ev))
                torch.cuda.synchronize()
                if it >= 2:
                    for (_, a), (n, b) in zip(ev[:-1], ev[1:]):
                        times.setdefault(n, []).append(a.elapsed_time(b))
            print("%3dx%-3d H%-2d %-4s rpb=%d " % (g, g, H, kind, rpb) +
                  " ".join("%s %.3f" % (n, sorted(t)[len(t) // 2]) for n, t in times.items()), flush=True)
