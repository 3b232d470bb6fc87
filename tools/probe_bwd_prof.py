"""Dev probe: per-role wait / work cycles of attn_bwd_kernel, averaged over
the CTAs and divided by the tiles each CTA ran.  Needs the HLA_BWD_PROF build:
  make VARIANT=bprof DEFS=-DHLA_BWD_PROF ; HLA_LIB_NAME=libhla_bprof.so python tools/probe_bwd_prof.py cfg2"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hla_synth
import paper_2511_05832_b200 as hla
from paper_2511_05832_b200 import _lib

CASES = {"cfg2": ("HWA", 64, 16, 16, 8), "cfg3": ("HSA", 64, 16, 16, 8), "cfg4": ("HNA", 128, 7, 16, 12),
         "dense2": ("DENSE", 64, 1, 16, 8), "cfg5s1": ("HWA", 64, 8, 128, 3, 32), "cfg5s2": ("HWA", 32, 8, 128, 6, 32),
         "cfg4b64": ("HNA", 128, 7, 16, 12, 64, 64), "hwt1": ("HWA", 56, 7, 128, 3, 32, 128, True),
         "hwt1s": ("HSWA", 56, 7, 128, 3, 32, 128, True)}
SLOTS = ["mma:ds_ready", "mma:epi_done", "mma:next_operands", "mma:dq_free", "mma:loop_total",
         "cmp:q_full", "cmp:s_full", "cmp:work", "cmp:rpb_flush", "dq:dq_full", "dq:drain", "dq:dkv_full", "dq:epilogue",
         "tma:kv_empty", "tma:q_empty", "-", "cmp:until_loads_done", "cmp:until_dS_done", "cmp:until_P_done",
         "cmp:until_p_ready"]
L = _lib.lib()
for name in (sys.argv[1:] or ["cfg2", "cfg3", "cfg4"]):
    kind, g, w, B, H = CASES[name][:5]
    d = CASES[name][5] if len(CASES[name]) > 5 else 64
    blk = CASES[name][6] if len(CASES[name]) > 6 else 128
    rpb = CASES[name][7] if len(CASES[name]) > 7 else False
    q, k, v, do = hla_synth.attention_inputs(B, g * g, H, d, device="cuda")
    lay = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, block=blk, device="cuda", rpb=rpb,
                                    shift=(w * w) // 2 if kind == "HSWA" else 0)
    for _ in range(3):
        lay.forward(q, k, v)
        lay.backward(do)
    torch.cuda.synchronize()
    buf = np.zeros((1024, 24), dtype=np.uint64)
    if name in ("cfg2", "dense2"):   # full-tile schedule
        n = L.hla_debug_bwd_prof(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), 148)
    else:                            # half-tile schedule (its own counters)
        n = L.hla_debug_bwd_split_prof(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), 148)
        name += " (half-tile schedule)"
    P = buf[:n].astype(np.float64)
    tiles = P[:, 15].sum()
    per = P[:, :20].sum(0) / max(tiles, 1)
    print("%s: %d tiles over %d CTAs; cycles per tile: %s" % (
        name, int(tiles), n, ", ".join("%s %.0f" % (s, x) for s, x in zip(SLOTS, per) if s[-1] != "-")), flush=True)
    del lay
