"""Dev probe: per-role wait / work cycles of attn_fwd_kernel, averaged over
the CTAs and divided by the kv-tiles each CTA ran.  Needs the HLA_FWD_PROF build:
  make VARIANT=fprof DEFS=-DHLA_FWD_PROF ; HLA_LIB_NAME=libhla_fprof.so python tools/probe_fwd_prof.py cfg2"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hla_synth
import paper_2511_05832_b200 as hla
from paper_2511_05832_b200 import _lib, api

CASES = {"cfg2": ("HWA", 64, 16, 16, 8), "cfg3": ("HSA", 64, 16, 16, 8), "cfg4": ("HNA", 128, 7, 16, 12),
         "dense2": ("DENSE", 64, 1, 16, 8), "cfg5s1": ("HWA", 64, 8, 128, 3, 32), "cfg5s2": ("HWA", 32, 8, 128, 6, 32)}
SLOTS = ["mma:s_free", "mma:poll_loop", "mma:loop_total", "sm:s_full", "sm:S_load", "sm:compute", "sm:pv_done",
         "sm:P_store", "sm:o_full", "sm:epilogue", "sm:epi+meta", "tma:o_staged", "tma:store_o", "tma:kv_empty",
         "-", "-", "-", "-", "-", "sm:s_full@t0", "-", "-", "-"]
L = _lib.lib()
for name in (sys.argv[1:] or ["cfg2", "cfg3", "cfg4"]):
    kind, g, w, B, H = CASES[name][:5]
    d = CASES[name][5] if len(CASES[name]) > 5 else 64
    q, k, v, do = hla_synth.attention_inputs(B, g * g, H, d, device="cuda")
    lay = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, device="cuda")
    s2c = None if os.environ.get("HLA_NO_GATHER") else lay.s2c
    lay.forward(q, k, v)
    for _ in range(3):   # the fused-reorder attention call of the layer (HLA_NO_GATHER=1: plain order)
        api.hla_attn_fwd(lay.desc, lay.mask, q, k, v, 0.0, lay.o, lay.lse, seq_to_cell=s2c)
    torch.cuda.synchronize()
    buf = np.zeros((1024, 24), dtype=np.uint64)
    n = L.hla_debug_fwd_prof(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), 296)
    P = buf[:n].astype(np.float64)
    tiles = P[:, 15].sum()
    per = P[:, :23].sum(0) / max(tiles, 1)
    span_ns = P[:, 18].max() - P[:, 17].min()
    cta_ns = (P[:, 18] - P[:, 17]).mean()
    mhz = (P[:, 16] / np.maximum(P[:, 18] - P[:, 17], 1)).mean() * 1e3
    print("%s: %d tiles over %d CTAs; span %.1f us, mean CTA %.1f us, start spread %.1f us, %.0f MHz; "
          "cycles per tile: %s" % (
              name, int(tiles), n, span_ns / 1e3, cta_ns / 1e3, (P[:, 17].max() - P[:, 17].min()) / 1e3, mhz,
              ", ".join("%s %.0f" % (s, x) for s, x in zip(SLOTS, per) if s != "-")), flush=True)
    dur = (P[:, 18] - P[:, 17]) / 1e3
    print("   per CTA: tiles min %d max %d, duration min %.1f max %.1f us" % (
        P[:, 15].min(), P[:, 15].max(), dur.min(), dur.max()), flush=True)
    for nt in sorted(set(P[:, 15].astype(int))):
        d = dur[P[:, 15] == nt]
        print("   %d tiles: %d CTAs, duration p0 %.1f p50 %.1f p100 %.1f us" % (nt, len(d), d.min(), np.median(d), d.max()))
    sm = P[:, 23].astype(int)
    tiles_sm = np.bincount(sm, weights=P[:, 15], minlength=148)
    end_sm = np.zeros(148)
    np.maximum.at(end_sm, sm, P[:, 18] - P[:, 17].min())
    print("   per SM: CTAs %s, tiles min %d max %d; SM end p0 %.1f p50 %.1f p100 %.1f us" % (
        np.bincount(np.bincount(sm, minlength=148)).tolist(), tiles_sm.min(), tiles_sm.max(),
        end_sm.min() / 1e3, np.median(end_sm) / 1e3, end_sm.max() / 1e3), flush=True)
    del lay
