#!/usr/bin/env python
"""bench.py -- Hilbert-guided local attention hot path on B200 (driver contract).

One STEP = one pass of the whole hot path over one batch, grid-order
tensors in and out, through the public HilbertLocalAttention API:
  block-sparse fwd (Hilbert gather of Q,K,V + scatter of O fused into the kernel) ;
  bwd preprocess (D, LSE2; gather of O,dO) ; block-sparse bwd (gathers, scatter of
  dK,dV) ; dQ finalize (+ inverse reorder)
(with HilbertLocalAttention(fused=False) the reorder runs as separate
hla_hilbert_perm passes instead, the paper's "Reshape" step).
The block mask and the Hilbert path are built once per shape, before timing
(the paper caches them).  Workload (N=1): BASELINE.json configs[1]
("cfg2": 64x64 grid, 8 heads, head_dim 64, HWA 256 tokens vs row-major 16x16
windows, block 128), batch 16 (the paper's batch).

metric "fwd+bwd ms ...": value = step time per batch of work for the whole job
= (max-over-ranks device time of one step) / (batches processed per step by all
ranks).  Each rank processes its own batch (weak scaling, no collective on the
hot path; NCCL only for the barrier and the max-reduction of timings).

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd ms and tensor-pipe % vs row-major + dense FA, 1/2/4/8 B200"
CONFIGS = {
    # name: Hilbert pattern, row-major baseline, grid side, window (cells), batch, heads, head_dim
    "cfg1": dict(kind="HWA", rm="WSA", grid=16, win=8, B=1, H=1, d=32,
                 text="16x16 grid, HWA 64 tokens vs WSA 8x8, 1 head, d32, batch 1"),
    "cfg2": dict(kind="HWA", rm="WSA", grid=64, win=16, B=16, H=8, d=64,
                 text="64x64 grid, HWA 256 tokens vs WSA 16x16, 8 heads, d64, block 128, batch 16"),
    "cfg3": dict(kind="HSA", rm="SA", grid=64, win=16, B=16, H=8, d=64,
                 text="64x64 grid, HSA 256 tokens vs SA 16x16, 8 heads, d64, block 128, batch 16"),
    "cfg4": dict(kind="HNA", rm="NA2D", grid=128, win=7, B=16, H=12, d=64,
                 text="128x128 grid, HNA 49 tokens vs NA2D 7x7, 12 heads, d64, block 128, batch 16"),
}
# cfg5: the HWT-T attention stack (SURVEY 8 cfg5 + 8(f) NEXT-1): Swin-T-like stages on the paper's
# feature-map sizes (generalized Hilbert path, ragged N), HWA / HSWA blocks alternating (HWT
# blocks come in pairs), each with HWT's global RPB, 7x7 = 49-token windows
STACK = {"cfg5": dict(B=128, d=32, stages=[(56, 3, 2, 7), (28, 6, 2, 7), (14, 12, 6, 7), (8, 24, 2, 8)],
                      text="HWT-T attention stack: stages 56x56/28x28/14x14/7x7->8x8 padded (N % 4 == 0 kernel "
                           "limit) (generalized Hilbert, ragged N), "
                           "heads 3/6/12/24, depths 2/2/6/2, B128, d32, 49-token windows (64 at the padded 8x8 stage), "
                           "HWA/HSWA alternating (shift = half a window), global RPB, block 128")}
# paper's row-major-block-sparse -> Hilbert fwd+bwd speedup on the nearest shape (RTX 3080)
PAPER_SPEEDUP = {"cfg2": (2.70, "WSA(Flex)->HWA 64x64 W8, P:L150-151"),
                 "cfg3": (1.62, "SA(Flex)->HSA 64x64 K9, P:L495-496"),
                 "cfg4": (1.58, "NA2D(Flex)->HNA 56x56 K7, P:L490-491")}
L2_FLUSH_BYTES = 512 << 20


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="cfg2", choices=sorted(CONFIGS) + sorted(STACK))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-variants", action="store_true", help="skip the row-major / dense comparison runs")
    p.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline leg")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


# ------------------------------------------------------------------ helpers
def bwd_bytes(T, d, mask):
    """Algorithmic HBM bytes of attn_bwd_kernel per launch: read Q, K, V, dO (8d per token-head),
    LSE, D (8); write dK, dV (4d); dQ: bf16 write (2d) for the q-blocks the dQ plan keeps
    local, one fp32 read + write of the accumulator (8d, TMA reduce-add) for the others."""
    mq = mask.row_ptr.numel() - 1
    nl = mq if mask.n_dq_nonlocal < 0 else mask.n_dq_nonlocal
    return int(T * (12 * d + 8) + T * (2 * d * (mq - nl) + 8 * d * nl) // mq)


def reduce_max_ms(ms, dist=None, device=None):
    """Max of a per-rank time over all ranks (the contract's max-over-ranks rule)."""
    import torch
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_value(step_ms, world):
    """Weak scaling: every rank processes one batch per step, so the whole job does
    `world` batches in step_ms (max over ranks) -> ms per batch of work."""
    return step_ms / world


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return {"hbm": pk["hbm_gbs"], "tf": pk["bf16_tflops"], "tf_sus": pk.get("bf16_tflops_sustained", pk["bf16_tflops"]),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm": 6650.0, "tf": 1590.0, "tf_sus": 1400.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """SM clock / throttle reasons sampled DURING the timed region (B200_PROFILING.md's
    clocks line).  NVML polled from a thread every ~1 ms (the timed region of a default
    run is only tens of ms, too short for `nvidia-smi -lms`); nvidia-smi as fallback."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._thread = None
        self._nvml = None

    def _poll(self):
        nv, h = self._nvml
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, attr in self.REASONS:
                    if mask & getattr(nv, attr, 0):
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.001)

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self._nvml = (nv, h)
        except Exception:
            self._nvml = None
            return
        self._thread = threading.Thread(target=self._poll, daemon=True)
        self._thread.start()

    def stop(self):
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=2)
        sms = [x for x in self.samples if x > 300]   # under load
        if not sms:
            return self._smi_once()
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(sms), "source": "nvml"}

    def _smi_once(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10).stdout
            sm, mx = [float(x) for x in out.strip().split(",")[:2]]
            return {"sm_mhz": sm, "sm_max_mhz": mx, "reasons": sorted(self.reasons), "samples": 1,
                    "source": "nvidia-smi after the timed region"}
        except Exception:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}


# ---------------------------------------------------------- oracle (CPU) leg
def oracle_step_sample(cfg, n_slices, seed=0):
    """The oracle as it stands on a bounded sample: Hilbert reorder (numpy
    indexing) + fp64 fwd+bwd of `n_slices` (b, h) slices.  Returns seconds."""
    import numpy as np

    import hla_synth
    from oracle import attention as oatt
    from oracle import hilbert as ohil
    from oracle.patterns import Spec
    g, B, H, d = cfg["grid"], cfg["B"], cfg["H"], cfg["d"]
    N = g * g
    spec = Spec(cfg["kind"], g, g, cfg["win"], cfg["win"])
    s2c, _ = ohil.hilbert_order(g, g)
    shape = (1, N, 1, d)
    t0 = time.perf_counter()
    for i in range(n_slices):
        q, k, v, do = (hla_synth.uniform_np(shape, seed + i, tid) for tid in (1, 2, 3, 4))
        qs, ks, vs, dos = (ohil.to_sequence(x, s2c)[0, :, 0].astype(np.float64) for x in (q, k, v, do))
        dQ, dK, dV, O, _ = oatt.attn_bwd_slice(qs, ks, vs, dos, spec, chunk=512)
        for x in (dQ, dK, dV, O):
            ohil.to_grid(x[None], s2c)
    return time.perf_counter() - t0


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(cfg, budget_s=15.0):
    slices_total = cfg["B"] * cfg["H"]
    t1 = oracle_step_sample(cfg, 1)
    n = int(max(1, min(slices_total, budget_s / max(t1, 1e-3))))
    t = oracle_step_sample(cfg, n, seed=1) if n > 1 else t1
    per_slice = t / n
    return {"value": round(per_slice * slices_total * 1e3, 3), "unit": "ms", "cores": blas_threads(),
            "kind": "oracle",
            "sample": "%d of %d (b,h) slices of one step (Hilbert reorder + fp64 fwd+bwd, numpy), "
                      "extrapolated x%d" % (n, slices_total, slices_total // max(n, 1))}


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    slices_total = cfg["B"] * cfg["H"]
    for _ in range(args.warmup):
        oracle_step_sample(cfg, 1)
    times = [oracle_step_sample(cfg, 1, seed=s) for s in range(args.steps)]
    ms = statistics.mean(times) * slices_total * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": round(ms, 3), "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (hla_synth)",
            "config": {"workload": args.config + ": " + cfg["text"], "global_batch": cfg["B"],
                       "seq_len": cfg["grid"] ** 2, "parallelism": "host cores (numpy BLAS)"},
            "cpu_baseline": {"value": round(ms, 3), "unit": "ms", "cores": blas_threads(), "kind": "oracle",
                             "sample": "each step = 1 of %d (b,h) slices (Hilbert reorder + fp64 fwd+bwd), "
                                       "extrapolated x%d" % (slices_total, slices_total)},
            "e2e": {"value": round(ms, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU leg
def run_stack(args):
    """--config cfg5: one step = fwd + bwd of every attention layer of the HWT-T stack."""
    import torch
    import torch.distributed as dist

    import hla_synth
    import paper_2511_05832_b200 as hla

    sc = STACK[args.config]
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    B, d = sc["B"], sc["d"]
    layers = []   # (layer, inputs) in execution order
    for si, (g, H, depth, w) in enumerate(sc["stages"]):
        N = g * g
        ins = hla_synth.attention_inputs(B, N, H, d, seed=100 * rank + si, device=dev)
        pair = [hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, shift=(w * w) // 2 if kind == "HSWA" else 0,
                                          device=dev, rpb=True) for kind in ("HWA", "HSWA")]
        gen = torch.Generator().manual_seed(si)
        for lay in pair:
            lay.rpb.copy_(torch.rand(lay.rpb.shape, generator=gen) * 2 - 1)
        for i in range(depth):
            layers.append((pair[i % 2], ins))
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    def one_step(rec=None):
        for lay, (q, k, v, do) in layers:
            lay.step(q, k, v, do, rec)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    def run(steps, marks):
        recs = []
        for _ in range(steps):
            flush.zero_()
            ev = [("start", torch.cuda.Event(enable_timing=True))]
            ev[0][1].record()

            def mark(name, ev=ev):
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ev.append((name, e))
            one_step(mark if marks else None)
            if not marks:
                mark("end")
            recs.append(ev)
        torch.cuda.synchronize()
        return recs

    # the step: one start / end event pair; the per-stage sums: a second, instrumented run
    sampler = ClockSampler(local)
    sampler.start()
    totals = run(args.steps, False)
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step = [ev[0][1].elapsed_time(ev[-1][1]) for ev in totals]
    per = {}
    for ev in run(args.steps, True):
        for (_, a), (name, b) in zip(ev[:-1], ev[1:]):
            per[name] = per.get(name, 0.0) + a.elapsed_time(b) / args.steps
    step_ms = reduce_max_ms(statistics.mean(step), dist if world > 1 else None, dev)
    peaks = load_peaks()
    # roofline of the stack's dominant kernel (sum over layers): algorithmic bytes / summed time
    tb = {"fwd": 0, "bwd": 0}
    for lay, (q, _, _, _) in layers:
        T = q.shape[0] * q.shape[1] * q.shape[2]
        tb["fwd"] += T * (8 * d + 4)
        tb["bwd"] += bwd_bytes(T, d, lay.mask)
    dom = max(("fwd", "bwd"), key=lambda kk: per[kk])
    ach = tb[dom] / (per[dom] * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm"], "unit": "GB/s",
            "frac": round(ach / peaks["hbm"], 4), "kernel": "attn_%s_kernel" % dom, "stage": dom,
            "share_of_step": round(per[dom] / statistics.mean(step), 4), "traffic": None,
            "note": "summed over the %d attention layers of the stack" % len(layers), "peak_source": peaks["source"]}
    line = {"metric": METRIC, "value": round(job_value(step_ms, world), 4), "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: hla_synth splitmix64 uniform, unit variance, bf16 (no dataset)",
            "config": {"workload": args.config + ": " + sc["text"], "global_batch": B * world,
                       "layers": len(layers), "parallelism": "dp%d" % world,
                       "l2": "flushed between timed steps (%d MiB write, untimed)" % (L2_FLUSH_BYTES >> 20)},
            "clocks": clocks, "e2e": None,
            "gpu_launches": sum(lay.launches_per_step for lay, _ in layers) * args.steps,
            "roofline": roof, "cpu_baseline": None,
            "breakdown_ms": {kk: round(vv, 4) for kk, vv in per.items()}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.config in STACK:
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "the oracle leg covers cfg1-cfg4 only"}))
            return
        run_stack(args)
        return
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    import hla_synth
    import paper_2511_05832_b200 as hla

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    peaks = load_peaks()

    g, B, H, d, win = cfg["grid"], cfg["B"], cfg["H"], cfg["d"], cfg["win"]
    N = g * g
    # each rank: its own batch shard (weak scaling); inputs resident in HBM before timing
    q, k, v, do = hla_synth.attention_inputs(B, N, H, d, seed=rank, device=dev)
    layer = hla.HilbertLocalAttention(cfg["kind"], g, g, win, win, B, H, d, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    def timed(lay, steps, warmup, with_marks=True, sampler=None):
        for _ in range(warmup):
            lay.step(q, k, v, do)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if sampler:
            sampler.start()
        rec = []
        for _ in range(steps):
            flush.zero_()                       # L2 flush between timed steps (untimed)
            ev = [("start", torch.cuda.Event(enable_timing=True))]
            ev[0][1].record()

            def mark(name, ev=ev):
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ev.append((name, e))
            lay.step(q, k, v, do, mark if with_marks else None)
            if not with_marks:
                mark("end")
            rec.append(ev)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clocks = sampler.stop() if sampler else None
        total = [ev[0][1].elapsed_time(ev[-1][1]) for ev in rec]
        stages = {}
        for ev in rec:
            for (_, a), (name, b) in zip(ev[:-1], ev[1:]):
                stages.setdefault(name, []).append(a.elapsed_time(b))
        # per-launch stages: median over the steps (robust to a single slow step)
        return total, {kk: statistics.median(vv) for kk, vv in stages.items()}, clocks

    sampler = ClockSampler(local)
    # the step is timed with one start / end event pair only; the per-kernel breakdown comes
    # from a second, instrumented run (one event after every launch: each intermediate event
    # adds ~2-3 us of GPU timeline, so it must not sit inside the headline measurement)
    total, _, clocks = timed(layer, args.steps, args.warmup, False, sampler)
    _, stages, _ = timed(layer, args.steps, 2, True)
    my_ms = statistics.mean(total)
    step_ms = reduce_max_ms(my_ms, dist if world > 1 else None, dev)
    value = job_value(step_ms, world)   # ms per batch of work for the whole job

    # --- row-major baseline and dense FA on the same shape (same kernels) ---
    variants = {}
    if not args.no_variants:
        vsteps = max(3, min(args.steps, 10))
        for name, kind in (("row_major", cfg["rm"]), ("dense", "DENSE")):
            lay = hla.HilbertLocalAttention(kind, g, g, win, win, B, H, d, device=dev)
            tot, _, _ = timed(lay, vsteps, 2, False)
            _, st, _ = timed(lay, vsteps, 1, True)
            variants[name] = {"pattern": kind, "ms_per_step": round(statistics.mean(tot), 4),
                              "fwd_ms": round(st["fwd"], 4), "bwd_ms": round(st["bwd_pre"] + st["bwd"] + st["bwd_fin"], 4),
                              "tiles_per_bh": lay.nnz}
            exec_flops = 14 * 128 * 128 * d * lay.nnz * B * H
            variants[name]["tensor_pct_executed"] = round(
                100 * exec_flops / ((st["fwd"] + st["bwd"]) * 1e-3) / (peaks["tf_sus"] * 1e12), 2)
            del lay
        # HWT's global relative position bias on the same layer (reading R19)
        lay = hla.HilbertLocalAttention(cfg["kind"], g, g, win, win, B, H, d, device=dev, rpb=True)
        lay.rpb.copy_(torch.rand(lay.rpb.shape, generator=torch.Generator().manual_seed(1)) * 2 - 1)
        tot, _, _ = timed(lay, vsteps, 2, False)
        _, st, _ = timed(lay, vsteps, 1, True)
        variants["global_rpb"] = {"pattern": cfg["kind"] + " + global RPB score_mod",
                                  "ms_per_step": round(statistics.mean(tot), 4), "fwd_ms": round(st["fwd"], 4),
                                  "bwd_ms": round(st["bwd_pre"] + st["bwd"] + st["bwd_fin"], 4)}
        del lay
        ours_attn = stages["fwd"] + stages["bwd_pre"] + stages["bwd"] + stages["bwd_fin"]
        rm = variants["row_major"]
        rm_attn = rm["fwd_ms"] + rm["bwd_ms"]
        variants["speedup_attn_vs_row_major"] = round(rm_attn / ours_attn, 3)
        variants["speedup_step_vs_row_major"] = round(rm["ms_per_step"] / step_ms, 3)
        variants["speedup_attn_vs_dense"] = round((variants["dense"]["fwd_ms"] + variants["dense"]["bwd_ms"]) / ours_attn, 3)
        if args.config in PAPER_SPEEDUP:
            variants["paper_speedup_fwd_bwd"] = {"value": PAPER_SPEEDUP[args.config][0],
                                                 "source": PAPER_SPEEDUP[args.config][1] + " (RTX 3080, context)"}

    # --- end to end through the public API: host -> device -> step -> host ---
    # Every step copies its inputs (Q, K, V, dO) from pinned host memory and reads its
    # results (O, dQ, dK, dV) back to pinned host memory inside the timed region.  The
    # copies run on two copy streams and the step on the compute stream, two steps in
    # flight (two layer instances = two sets of device buffers): step i+1's host->device
    # copies overlap step i's compute and device->host copies (full-duplex link).
    e2e = None
    if not args.no_e2e:
        hin = [x.cpu().pin_memory() for x in (q, k, v, do)]
        layers = [layer, hla.HilbertLocalAttention(cfg["kind"], g, g, win, win, B, H, d, device=dev)]
        din = [[torch.empty_like(x) for x in (q, k, v, do)] for _ in range(2)]
        hout = [[torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in (q, q, q, q)] for _ in range(2)]
        s_in, s_out, s_cmp = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.current_stream(dev)
        ev_free = [None, None]

        def e2e_step(i):
            j = i % 2
            with torch.cuda.stream(s_in):
                if ev_free[j] is not None:
                    s_in.wait_event(ev_free[j])       # slot j's buffers: step i-2 fully read back
                for dst, src in zip(din[j], hin):
                    dst.copy_(src, non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_in)
            s_cmp.wait_event(ev_in)
            o = layers[j].forward(*din[j][:3])
            ev_o = torch.cuda.Event()
            ev_o.record(s_cmp)
            grads = layers[j].backward(din[j][3])
            ev_g = torch.cuda.Event()
            ev_g.record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_o)
                hout[j][0].copy_(o, non_blocking=True)
                s_out.wait_event(ev_g)
                for dst, src in zip(hout[j][1:], grads):
                    dst.copy_(src, non_blocking=True)
                ev_free[j] = torch.cuda.Event()
                ev_free[j].record(s_out)

        esteps = max(4, min(args.steps, 10))
        for i in range(2):                          # warm-up (untimed)
            e2e_step(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_in)
        for i in range(2, 2 + esteps):
            e2e_step(i)
        s_out.wait_stream(s_cmp)
        e1.record(s_out)
        torch.cuda.synchronize()
        te = reduce_max_ms(e0.elapsed_time(e1) / esteps, dist if world > 1 else None, dev)
        nbytes = sum(x.numel() * x.element_size() for x in hin)
        e2e = {"value": round(job_value(te, world), 4), "unit": "ms", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "steps": esteps,
               "path": "pinned host -> (copy stream) -> HilbertLocalAttention.forward/backward (compute stream) -> "
                       "(copy stream) -> pinned host; two steps in flight (double-buffered device tensors)"}

    # --- roofline of the dominant kernel (share of the step) ---
    T = B * H * N                               # token-heads per launch
    tiles = layer.nnz * B * H
    kern = {
        "fwd": {"bytes": T * (8 * d + 4), "flops": 4 * 128 * 128 * d * tiles, "name": "attn_fwd_kernel"},
        "bwd": {"bytes": bwd_bytes(T, d, layer.mask), "flops": 10 * 128 * 128 * d * tiles, "name": "attn_bwd_kernel"},
        "perm_qkv": {"bytes": 3 * 2 * T * d * 2, "flops": 0, "name": "hilbert_perm_kernel"},
        "perm_grads": {"bytes": 3 * 2 * T * d * 2, "flops": 0, "name": "hilbert_perm_kernel"},
    }
    dom = max((kk for kk in kern if kk in stages), key=lambda kk: stages[kk])
    ms_dom = stages[dom]
    kd = kern[dom]
    ridge = peaks["tf_sus"] * 1e12 / (peaks["hbm"] * 1e9)
    ai = kd["flops"] / kd["bytes"] if kd["bytes"] else 0
    if ai < ridge:
        ach = kd["bytes"] / (ms_dom * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm"], "unit": "GB/s",
                "frac": round(ach / peaks["hbm"], 4)}
    else:
        ach = kd["flops"] / (ms_dom * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": round(ach, 1), "peak": peaks["tf_sus"], "unit": "TFLOP/s",
                "frac": round(ach / peaks["tf_sus"], 4)}
    roof.update({"kernel": kd["name"], "stage": dom, "share_of_step": round(ms_dom / my_ms, 4),
                 "ms_per_launch": round(ms_dom, 5), "algorithmic_bytes_per_launch": kd["bytes"],
                 "algorithmic_flops_per_launch": kd["flops"], "arith_intensity": round(ai, 1),
                 "peak_source": peaks["source"], "traffic": None})
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(args.config, {}).get(dom)
        if tr:
            roof["traffic"] = tr
    except Exception:
        pass

    attn_ms = stages["fwd"] + stages["bwd_pre"] + stages["bwd"] + stages["bwd_fin"]
    exec_flops = 14 * 128 * 128 * d * tiles
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg)

    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: hla_synth splitmix64 uniform, unit variance, bf16 (no dataset)",
        "config": {"workload": args.config + ": " + cfg["text"], "global_batch": B * world, "seq_len": N,
                   "parallelism": "dp%d (batch shards, no collective on the hot path)" % world,
                   "l2": "flushed between timed steps (%d MiB write, untimed)" % (L2_FLUSH_BYTES >> 20),
                   "step": ("fwd+bwd_pre+bwd+bwd_fin (Hilbert reorder fused into the kernels)" if layer.fused else
                            "perm(qkv)+fwd+perm(o)+perm(dO)+bwd_pre+bwd+bwd_fin+perm(dq,dk,dv)"),
                   "mask": "built once before timing (%d of %d tiles per (b,h) executed)" % (layer.nnz, (N // 128) ** 2),
                   "timing": "CUDA events: one start/end pair per step (value = mean); breakdown_ms = per-launch "
                             "medians from a second run with one event after every launch"},
        "clocks": clocks, "e2e": e2e, "gpu_launches": layer.launches_per_step * args.steps,
        "roofline": roof, "cpu_baseline": cpu,
        "breakdown_ms": {kk: round(vv, 5) for kk, vv in stages.items()},
        "attn_ms": round(attn_ms, 4),
        "tensor_pct_executed": round(100 * exec_flops / (attn_ms * 1e-3) / (peaks["tf_sus"] * 1e12), 2),
        "variants": variants,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
