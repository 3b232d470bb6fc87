"""Dev probe: Hilbert order (gather4 loads) vs the tiled Hilbert order (include/hla.h
HLA_ORDER_HILBERT_TILED: 8-row TMA boxes at d = 32), same layer shapes, same process; CUDA-event
timed fwd / bwd (warm L2) and the max relative error of both against a dense fp32 torch reference.
  python tools/probe_box8.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import hla_synth
import paper_2511_05832_b200 as hla

CASES = [("cfg2", 64, 16, 16, 8, 64, 128), ("cfg5s1", 64, 8, 128, 3, 32, 64), ("cfg5s2", 32, 8, 128, 6, 32, 64),
         ("cfg5s1b128", 64, 8, 128, 3, 32, 128)]


def ref_slice(q, k, v, do, wid, scale):
    q, k, v, do = (t.float().requires_grad_(True) for t in (q, k, v, do))
    s = (q @ k.t()) * scale
    s = s.masked_fill(wid[:, None] != wid[None, :], float("-inf"))
    o = torch.softmax(s, -1) @ v
    o.backward(do)
    return o.detach(), q.grad, k.grad, v.grad


for (name, g, w, B, H, d, blk), box8 in [(c, t) for c in CASES for t in (False, True)]:
    N = g * g
    q, k, v, do = hla_synth.attention_inputs(B, N, H, d, device="cuda")
    lay = hla.HilbertLocalAttention("HWA", g, g, w, w, B, H, d, block=blk, device="cuda", tiled=box8)
    s2c, _ = hla.hla_hilbert_index(g, g)
    c2s = torch.empty_like(s2c)
    c2s[s2c.long()] = torch.arange(N, device="cuda", dtype=s2c.dtype)
    wid = (c2s // (w * w)).long()
    for _ in range(3):
        lay.forward(q, k, v)
        lay.backward(do)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf = tb = 0.0
    R = 20
    for _ in range(R):
        ev[0].record()
        o = lay.forward(q, k, v)
        ev[1].record()
        dq, dk, dv = lay.backward(do)
        ev[2].record()
        torch.cuda.synchronize()
        tf += ev[0].elapsed_time(ev[1])
        tb += ev[1].elapsed_time(ev[2])
    err = []
    for b, h in [(0, 0), (B - 1, H - 1)]:
        ro, rq, rk, rv = ref_slice(q[b, :, h], k[b, :, h], v[b, :, h], do[b, :, h], wid, d ** -0.5)
        for got, ref in ((o, ro), (dq, rq), (dk, rk), (dv, rv)):
            e = (got[b, :, h].float() - ref).abs().max().item() / max(ref.abs().max().item(), 1e-6)
            err.append(e)
    print("%s %s: fwd %.1f us, bwd %.1f us, max rel err %.4f" % ("box8" if box8 else "gather4", name,
                                                               1e3 * tf / R, 1e3 * tb / R, max(err)), flush=True)
    del lay
