"""Small hot-path workloads for compute-sanitizer (SURVEY 4.2 tier T3): cfg1 (HWA 16x16, d32) and
one (b, h) slice of cfg2 / cfg3 shapes (64x64, d64; HWA full tiles, HSA partial tiles), forward +
backward through the public layer, plus the explicit permutation path and the block-mask builder."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hla_synth
import paper_2511_05832_b200 as hla

dev = "cuda"
cases = [("HWA", 16, 8, 1, 1, 32, True), ("HWA", 64, 16, 1, 1, 64, True), ("HSA", 64, 16, 1, 1, 64, True),
         ("HWA", 64, 16, 1, 1, 64, False)]
for kind, g, w, B, H, d, fused in cases:
    q, k, v, do = (t.to(dev) for t in hla_synth.attention_inputs(B, g * g, H, d, seed=0))
    layer = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, device=dev, fused=fused)
    o = layer.forward(q, k, v)
    dq, dk, dv = layer.backward(do)
    torch.cuda.synchronize()
    assert torch.isfinite(o.float()).all() and torch.isfinite(dq.float()).all()
    print("ok", kind, g, d, "fused" if fused else "explicit perm", flush=True)
# r05: the paths added since r03 -- global RPB score_mod (fwd + table gradient, d32 / d64), HSWA
# (shifted windows, all-partial tiles), HNA (clamped neighbourhoods, dQ accumulator + finalize),
# and the generalized Hilbert curve on a non-2^k grid (56x56, ragged last tile)
cases2 = [("HWA", 64, 16, 1, 2, 64, False), ("HWA", 56, 7, 1, 1, 32, True), ("HSWA", 32, 8, 2, 3, 32, True),
          ("HNA", 32, 5, 1, 2, 64, False), ("HSWA", 8, 8, 2, 2, 32, True)]
for kind, g, w, B, H, d, rpb in cases2:
    q, k, v, do = (t.to(dev) for t in hla_synth.attention_inputs(B, g * g, H, d, seed=1))
    shift = (w * w) // 2 if kind == "HSWA" else 0
    layer = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, shift=shift, device=dev, rpb=rpb)
    if rpb:
        layer.rpb.uniform_(-1, 1)
    o = layer.forward(q, k, v)
    dq, dk, dv = layer.backward(do)
    torch.cuda.synchronize()
    assert torch.isfinite(o.float()).all() and torch.isfinite(dq.float()).all()
    assert not rpb or torch.isfinite(layer.drpb).all()
    print("ok", kind, g, d, "rpb" if rpb else "no rpb", flush=True)
