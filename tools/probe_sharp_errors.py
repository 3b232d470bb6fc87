"""Dev probe (reading R16): GPU vs fp64-oracle error of the backward on the sharp
stress input, beside the error of the bf16 rounding model (tests/parity.py) -- max, p99.9, mean."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import torch

import hla_synth
import paper_2511_05832_b200 as hla
from oracle import attention as oatt
from oracle.patterns import Spec
from parity import emulated_slice, to_np
from test_gpu_attention import SMALL

for kind, gh, gw, wh, ww, B, H, d in SMALL:
    shift = (wh * ww) // 2 if kind == "HSWA" else 0
    N = gh * gw
    q, k, v, do = [t.to("cuda") for t in hla_synth.attention_inputs(B, N, H, d, seed=7, sharp=True)]
    desc = hla.pattern_desc(kind, gh, gw, wh, ww, shift=shift)
    m = hla.hla_build_block_mask(desc, "cuda")
    o, lse = hla.hla_attn_fwd(desc, m, q, k, v)
    dq, dk, dv = hla.hla_attn_bwd(desc, m, q, k, v, o, lse, do)
    torch.cuda.synchronize()
    spec = Spec(kind, gh, gw, wh, ww, shift=shift)
    dQ, dK, dV = oatt.attn_bwd(to_np(q), to_np(k), to_np(v), to_np(do), spec)
    emu = [np.zeros_like(dQ), np.zeros_like(dK), np.zeros_like(dV)]
    for b in range(B):
        for h in range(H):
            r = emulated_slice(*(to_np(t[b, :, h]) for t in (q, k, v, do)), spec)
            for i in range(3):
                emu[i][b, :, h] = r[i + 1]
    out = []
    for name, got, ref, e in (("dQ", dq, dQ, emu[0]), ("dK", dk, dK, emu[1]), ("dV", dv, dV, emu[2])):
        eg, ee = np.abs(to_np(got) - ref), np.abs(e - ref)
        out.append("%s max %.4f/%.4f p999 %.4f/%.4f mean %.5f/%.5f" % (
            name, eg.max(), ee.max(), np.quantile(eg, 0.999), np.quantile(ee, 0.999), eg.mean(), ee.mean()))
    print("%-5s %dx%d w%dx%d d%d | %s" % (kind, gh, gw, wh, ww, d, " | ".join(out)), flush=True)
