#!/usr/bin/env python
"""bench.py -- Hilbert-guided local attention hot path on B200 (driver contract).

One STEP = one pass of the whole hot path over one global batch, grid-order
tensors in and out, through the public HilbertLocalAttention API:
  block-sparse fwd (Hilbert gather of Q,K,V + scatter of O fused into the kernel) ;
  bwd preprocess (D, LSE2; gather of O,dO) ; block-sparse bwd (gathers, scatter of
  dK,dV) ; dQ finalize (+ inverse reorder)
(HilbertLocalAttention(fused=False) runs the reorder as separate hla_hilbert_perm passes
instead, the paper's "Reshape" step; that variant is timed too, for perm_ms).
The block mask and the Hilbert path are built once per shape, before timing (the paper
caches them); their build time is reported separately (mask_build_ms).
Workload (N=1): BASELINE.json configs[1] ("cfg2": 64x64 grid, 8 heads, head_dim 64, HWA
256 tokens vs row-major 16x16 windows, block 128), batch 16 (the paper's batch).

Multi-GPU (north_star "partitioned across the 8xB200 box by batch x head"):
STRONG scaling at the fixed global batch.  plan_shards() gives every rank a contiguous
block of (batch, head) units -- B/g whole batches, or head groups of one batch when B < g;
the units are independent (no exchange step), so there is no collective on the hot path.
NCCL carries only the barrier, the max-reduction of step times and, after the timed loop,
the all_gather of per-rank statistics (times, units, backward-invariant residuals).
value = max-over-ranks device time of one step of the whole global batch.

`python bench.py --gpus N` outside torchrun re-executes itself under
torch.distributed.run with N ranks; under torchrun WORLD_SIZE must equal --gpus.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]
"""

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
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
                 text="64x64 grid, HWA 256 tokens vs WSA 16x16, 8 heads, d64, batch 16"),
    "cfg3": dict(kind="HSA", rm="SA", grid=64, win=16, B=16, H=8, d=64,
                 text="64x64 grid, HSA 256 tokens vs SA 16x16, 8 heads, d64, batch 16"),
    "cfg4": dict(kind="HNA", rm="NA2D", grid=128, win=7, B=16, H=12, d=64,
                 text="128x128 grid, HNA 49 tokens vs NA2D 7x7, 12 heads, d64, batch 16"),
}
# attention stacks of a Hilbert Window Transformer (HWT-T: Swin-T stage shapes)
#   cfg5     BASELINE.json configs[4] as stated: 56/28/14/7 grids padded to the Hilbert grid
#            64/32/16/8, window 49 -> 64 tokens (8 x 8), heads 3/6/12/24, batch 128, all HWA
#            (MVP), depths 2/2/6/2, d32
#   cfg5-hwt the HWT-T stack itself: unpadded 56/28/14 grids on the
#            generalized Hilbert curve (ragged N; 7x7 -> 8x8 padded: the kernels need N % 4 == 0),
#            49-token windows, HWA / HSWA alternating (shift = half a window), global RPB
STACK = {
    "cfg5": dict(B=128, d=32, block=64, hswa=False, rpb=False,
                 stages=[(64, 3, 2, 8), (32, 6, 2, 8), (16, 12, 6, 8), (8, 24, 2, 8)],
                 text="HWT-T attention stack as BASELINE states it: 56x56/28x28/14x14/7x7 padded to "
                      "64x64/32x32/16x16/8x8 Hilbert grids, windows 49->64 tokens (8x8), heads 3/6/12/24, "
                      "depths 2/2/6/2, all HWA, B128, d32"),
    "cfg5-hwt": dict(B=128, d=32, block=128, hswa=True, rpb=True,
                     stages=[(56, 3, 2, 7), (28, 6, 2, 7), (14, 12, 6, 7), (8, 24, 2, 8)],
                     text="HWT-T attention stack: stages 56x56/28x28/14x14 (generalized Hilbert, ragged N) "
                          "and 7x7->8x8 padded, heads 3/6/12/24, depths 2/2/6/2, B128, d32, 49-token windows "
                          "(64 at 8x8), HWA/HSWA alternating (shift = half a window), global RPB"),
}
# paper's row-major-block-sparse -> Hilbert fwd+bwd speedup on the nearest shape (RTX 3080)
PAPER_SPEEDUP = {"cfg2": (2.70, "WSA(Flex)->HWA 64x64 W8, P:L150-151"),
                 "cfg3": (1.62, "SA(Flex)->HSA 64x64 K9, P:L495-496"),
                 "cfg4": (1.58, "NA2D(Flex)->HNA 56x56 K7, P:L490-491")}
# the paper's headline speedups, with their hardware (context, not targets)
PAPER_HEADLINES = {
    "window_about_4x": "dense WSA 2.74 ms / HWA(Flex) 0.68 ms, forward, 128x128 grid, 16x16 windows, "
                       "RTX 3080 (P:L7, P:L161-163, P:L167)",
    "slide_about_18x": "naive SA 5.85 ms / HSA(Flex) 0.32 ms, forward, 56x56 grid, 7x7 kernel, "
                       "RTX 3080 (P:L7, P:L226-228)",
}
PAPER_TIMING = ("the paper: mean of 10 runs x 100 iterations, first 25% warm-up (P:L137); here: W warm-up "
                "steps then K timed steps (driver contract)")
L2_FLUSH_BYTES = 512 << 20


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="cfg2", choices=sorted(CONFIGS) + sorted(STACK))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--block", type=int, default=None, choices=[64, 128],
                   help="tile block b_q = b_k (default: the config's; SURVEY 8: 128, cfg5 64)")
    p.add_argument("--no-variants", action="store_true", help="skip the row-major / dense / RPB / unfused runs")
    p.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline leg")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args(argv)


# ------------------------------------------------------------------ multi-GPU plumbing
def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_ranks(args, argv):
    """--gpus N > 1 outside torchrun: re-execute under torch.distributed.run with N ranks
    (one process per GPU, rendezvous on 127.0.0.1).  Returns the exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


def plan_shards(B, H, world):
    """Strong-scaling partition of the B x H independent (batch, head) attention units over
    `world` ranks: rank r gets the contiguous block (b0, b1, h0, h1) --
    B / world whole batches when world divides B; when B < world and world / B divides H,
    each batch's heads are split into world / B contiguous groups.  Every unit belongs to
    exactly one rank.  None: no such partition (the config runs as replicas)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if B % world == 0:
        k = B // world
        return [(r * k, (r + 1) * k, 0, H) for r in range(world)]
    if world % B == 0 and H % (world // B) == 0:
        g = world // B
        hk = H // g
        return [(r // g, r // g + 1, (r % g) * hk, (r % g + 1) * hk) for r in range(world)]
    return None


def reduce_max_ms(ms, dist=None, device=None):
    """Max of a per-rank time over all ranks (the contract's max-over-ranks rule)."""
    import torch
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rank_stats(values, dist=None, device=None):
    """all_gather of a fixed-length list of floats from every rank (after the timed loop;
    NCCL on the GPU box, gloo in the CPU tests) -> list indexed by rank."""
    import torch
    t = torch.tensor([float(x) for x in values], dtype=torch.float64, device=device)
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return [t.tolist()]
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.tolist() for o in out]


# ------------------------------------------------------------------ helpers
def bwd_bytes(T, d, mask, fused_pre=False):
    """Algorithmic HBM bytes of the backward main kernel per launch: read Q, K, V, dO (8d per
    token-head), LSE, D (8); write dK, dV (4d); dQ: bf16 write (2d) for the q-blocks the dQ
    plan keeps local, one fp32 read + write of the accumulator (8d, TMA reduce-add) for the others.
    fused_pre (preprocess folded into the kernel): read O (2d) and the raw LSE (4) instead of
    LSE, D (8): T (14d + 4) + the dQ part (all local: T (16d + 4))."""
    mq = mask.row_ptr.numel() - 1
    nl = mq if mask.n_dq_nonlocal < 0 else mask.n_dq_nonlocal
    if fused_pre:   # O (2d) and the raw LSE (4) instead of LSE, D (8); dQ as above
        return int(T * (14 * d + 4) + T * (2 * d * (mq - nl) + 8 * d * nl) // mq)
    return int(T * (12 * d + 8) + T * (2 * d * (mq - nl) + 8 * d * nl) // mq)


def exec_flops(tiles, d, block=128):
    """Tensor-core flops on EXECUTED tiles of one fwd+bwd: 4 b^2 d (S, PV) + 10 b^2 d (S, dP,
    dV, dK, dQ recomputed / computed in the backward) per tile; empty tiles are never counted."""
    return 14 * block * block * d * tiles


def tensor_pct(flops, ms, peak_tf):
    """Executed-tile tensor throughput as % of the peak -- the same definition for the headline
    and every variant: flops / (fwd + bwd_pre + bwd + bwd_fin time)."""
    return round(100 * flops / (ms * 1e-3) / (peak_tf * 1e12), 2)


def _ncu_traffic(key, stage):
    """DRAM bytes per launch of the stage's kernel from the committed ncu launch lists
    (profiles/ncu_traffic.json; dram__bytes_read.sum + dram__bytes_write.sum), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(key, {}).get(stage)
    except Exception:
        return None


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
    g, d = cfg["grid"], cfg["d"]
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
            "kind": "oracle", "measured_s": round(t, 3), "slices_measured": n, "slices_per_step": slices_total,
            "sample": "%d of %d (b,h) slices of one step (Hilbert reorder + fp64 fwd+bwd, numpy), measured %.2f s, "
                      "extrapolated x%.2f" % (n, slices_total, t, slices_total / n)}


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
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (hla_synth)",
            "config": {"workload": args.config + ": " + cfg["text"], "global_batch": cfg["B"],
                       "seq_len": cfg["grid"] ** 2, "parallelism": "host cores (numpy BLAS), rank 0 only"},
            "cpu_baseline": {"value": round(ms, 3), "unit": "ms", "cores": blas_threads(), "kind": "oracle",
                             "measured_s_per_slice": [round(t, 4) for t in times],
                             "sample": "each step = 1 of %d (b,h) slices (Hilbert reorder + fp64 fwd+bwd) measured "
                                       "(mean %.3f s), extrapolated x%d to the whole step"
                                       % (slices_total, statistics.mean(times), slices_total)},
            "e2e": {"value": round(ms, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU leg
def _timed(step, steps, warmup, flush=None, marks=True, sampler=None, dist=None, world=1):
    """Device-timed steps: one start/end CUDA-event pair per step (marks=False), or an event
    after every launch for the per-launch breakdown (marks=True).  flush: L2 flush buffer
    written between steps (untimed); None = warm L2."""
    import torch
    for _ in range(warmup):
        step(None)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
    rec = []
    for _ in range(steps):
        if flush is not None:
            flush.zero_()
        ev = [("start", torch.cuda.Event(enable_timing=True))]
        ev[0][1].record()

        def mark(name, ev=ev):
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            ev.append((name, e))
        step(mark if marks else None)
        if not marks:
            mark("end")
        rec.append(ev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    total = [ev[0][1].elapsed_time(ev[-1][1]) for ev in rec]
    stages, sums = {}, {}
    for ev in rec:
        for (_, a), (name, b) in zip(ev[:-1], ev[1:]):
            stages.setdefault(name, []).append(a.elapsed_time(b))
            sums[name] = sums.get(name, 0.0) + a.elapsed_time(b) / steps
    # per-launch medians (single-layer steps) and, per launch name, the mean over steps of its
    # summed time within a step (the stacks: the same name recurs once per layer)
    return total, {kk: statistics.median(vv) for kk, vv in stages.items()}, sums, clocks


def _init_dist(args):
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit("bench.py: WORLD_SIZE=%d but --gpus %d (launch one process per GPU)" % (world, args.gpus))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    return rank, world, local, dev, dist


def invariant_residuals(dk, dv, do):
    """Backward invariants of every (b, h) slice: sum_k dK[k] = 0 and
    sum_k dV[k] = sum_q dO[q] (exact for the fp64 oracle; softmax rows sum to one).  Returns
    (max |sum dK|, max |sum dV - sum dO|, bound) -- bound = the bf16 rounding allowance the
    GPU parity tests use, 8 sqrt(N) rms(dK) 2^-8."""
    N = dk.shape[1]
    rk = float(dk.float().sum(1).abs().max())
    rv = float((dv.float().sum(1) - do.float().sum(1)).abs().max())
    bound = 8 * math.sqrt(N) * float(dk.float().pow(2).mean().sqrt()) * 2 ** -8
    return rk, rv, bound


def run_stack(args):
    """--config cfg5 / cfg5-hwt: one step = fwd + bwd of every attention layer of the HWT-T stack."""
    import torch

    import hla_synth
    import paper_2511_05832_b200 as hla

    sc = STACK[args.config]
    blk = args.block or sc["block"]
    rank, world, local, dev, dist = _init_dist(args)
    B, d = sc["B"], sc["d"]
    if B % world:
        raise SystemExit("cfg5 stacks shard their batch of %d over the ranks: %d does not divide it" % (B, world))
    b0, b1 = rank * B // world, (rank + 1) * B // world
    layers = []   # (layer, inputs) in execution order
    for si, (g, H, depth, w) in enumerate(sc["stages"]):
        N = g * g
        ins = hla_synth.attention_inputs_block(B, N, H, d, b0, b1, 0, H, seed=100 + si, device=dev)
        kinds = ("HWA", "HSWA") if sc["hswa"] else ("HWA",)
        pair = [hla.HilbertLocalAttention(kind, g, g, w, w, b1 - b0, H, d, block=blk,
                                          shift=(w * w) // 2 if kind == "HSWA" else 0, device=dev, rpb=sc["rpb"])
                for kind in kinds]
        gen = torch.Generator().manual_seed(si)
        for lay in pair:
            if sc["rpb"]:
                lay.rpb = torch.rand(lay.rpb.shape, generator=gen) * 2 - 1
        for i in range(depth):
            layers.append((pair[i % len(pair)], ins))
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    def one_step(rec=None):
        for lay, (q, k, v, do) in layers:
            lay.step(q, k, v, do, rec)

    sampler = ClockSampler(local)
    totals, _, _, clocks = _timed(one_step, args.steps, args.warmup, flush, False, sampler, dist, world)
    # per-stage sums over the layers: a second, instrumented run (events after every launch)
    _, _, per, _ = _timed(one_step, args.steps, 1, flush, True, None, dist, world)
    my_ms = statistics.mean(totals)
    step_ms = reduce_max_ms(my_ms, dist if world > 1 else None, dev)
    ranks = gather_rank_stats([rank, b1 - b0, my_ms], dist if world > 1 else None, dev)
    peaks = load_peaks()
    # roofline of the stack's dominant kernel (summed over the layers): algorithmic bytes / summed time
    tb = {"fwd": 0, "bwd": 0}
    for lay, (q, _, _, _) in layers:
        T = q.shape[0] * q.shape[1] * q.shape[2]
        tb["fwd"] += T * (8 * d + 4)
        tb["bwd"] += bwd_bytes(T, d, lay.mask, lay.fused_bwd)
    dom = max(("fwd", "bwd"), key=lambda kk: per.get(kk, 0.0))
    ach = tb[dom] / (per[dom] * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm"], "unit": "GB/s",
            "frac": round(ach / peaks["hbm"], 4), "kernel": "attn_%s_kernel" % dom, "stage": dom,
            "share_of_step": round(per[dom] / my_ms, 4),
            "traffic": (lambda t: t * len(layers) if t and world == 1 else None)(
                _ncu_traffic(args.config + ("@64" if blk == 64 else ""), dom)),
            "note": "summed over the %d attention layers of the stack (rank 0)" % len(layers),
            "peak_source": peaks["source"]}
    line = {"metric": METRIC, "value": round(step_ms, 4), "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: hla_synth splitmix64 uniform, unit variance, bf16 (no dataset)",
            "config": {"workload": "%s: %s, block %d" % (args.config, sc["text"], blk), "global_batch": B,
                       "layers": len(layers), "block": blk,
                       "parallelism": "batch shards: rank r runs batches [r B/%d, (r+1) B/%d), all heads" % (world, world),
                       "l2": "flushed between timed steps (%d MiB write, untimed)" % (L2_FLUSH_BYTES >> 20),
                       "timing": PAPER_TIMING},
            "clocks": clocks, "e2e": None,
            "gpu_launches": sum(lay.launches_per_step for lay, _ in layers) * args.steps,
            "roofline": roof, "cpu_baseline": None,
            "breakdown_ms": {kk: round(vv, 4) for kk, vv in per.items()},
            "ranks": [{"rank": int(r[0]), "batches": int(r[1]), "step_ms": round(r[2], 4)} for r in ranks]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_single(args):
    import torch

    import hla_synth
    import paper_2511_05832_b200 as hla

    cfg = CONFIGS[args.config]
    blk = args.block or 128
    rank, world, local, dev, dist = _init_dist(args)
    peaks = load_peaks()
    g, B, H, d, win = cfg["grid"], cfg["B"], cfg["H"], cfg["d"], cfg["win"]
    N = g * g
    plan = plan_shards(B, H, world)
    b0, b1, h0, h1 = plan[rank] if plan else (0, B, 0, H)
    Bs, Hs = b1 - b0, h1 - h0
    # this rank's shard of the global batch (exactly the global tensors' values), resident in HBM
    q, k, v, do = hla_synth.attention_inputs_block(B, N, H, d, b0, b1, h0, h1, seed=0, device=dev)

    # mask build (once per shape, outside the step; reported separately): host wall time of
    # hla_build_block_mask + the bwd plan, both synchronous
    builds = []
    for _ in range(3):
        t0 = time.perf_counter()
        hla.hla_build_block_mask(hla.pattern_desc(cfg["kind"], g, g, win, win, block=blk), dev)
        builds.append((time.perf_counter() - t0) * 1e3)
    layer = hla.HilbertLocalAttention(cfg["kind"], g, g, win, win, Bs, Hs, d, block=blk, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    step = lambda mark, lay=layer: lay.step(q, k, v, do, mark)   # noqa: E731

    sampler = ClockSampler(local)
    # the step is timed with one start / end event pair only; the per-kernel breakdown comes
    # from a second, instrumented run (one event after every launch: each intermediate event
    # adds ~2-3 us of GPU timeline, so it must not sit inside the headline measurement)
    total, _, _, clocks = _timed(step, args.steps, args.warmup, flush, False, sampler, dist, world)
    _, stages, _, _ = _timed(step, args.steps, 2, flush, True, None, dist, world)
    warm, _, _, _ = _timed(step, args.steps, 2, None, False, None, dist, world)
    my_ms = statistics.mean(total)
    step_ms = reduce_max_ms(my_ms, dist if world > 1 else None, dev)
    warm_ms = reduce_max_ms(statistics.mean(warm), dist if world > 1 else None, dev)
    dq, dk, dv = layer.step(q, k, v, do)
    torch.cuda.synchronize()
    rk, rv, rbound = invariant_residuals(dk, dv, do)

    tiles = layer.tiles * Bs * Hs   # executed 128 x 128 tiles (block 64: windows)
    attn_ms = stages["fwd"] + stages.get("bwd_pre", 0.0) + stages["bwd"] + stages.get("bwd_fin", 0.0)

    # --- variants on this rank's shard (same kernels): row-major baseline, dense FA, HWT's
    #     global RPB, and the unfused reorder (explicit hla_hilbert_perm passes: perm_ms) ---
    variants, perm = {}, None
    if not args.no_variants:
        vsteps = max(3, min(args.steps, 10))
        for name, kind in (("row_major", cfg["rm"]), ("dense", "DENSE")):
            lay = hla.HilbertLocalAttention(kind, g, g, win, win, Bs, Hs, d, block=blk, device=dev)
            st_fn = lambda mark, lay=lay: lay.step(q, k, v, do, mark)   # noqa: E731
            tot, _, _, _ = _timed(st_fn, vsteps, 2, flush, False, None, dist, world)
            _, st, _, _ = _timed(st_fn, vsteps, 1, flush, True, None, dist, world)
            a_ms = st["fwd"] + st.get("bwd_pre", 0.0) + st["bwd"] + st.get("bwd_fin", 0.0)
            variants[name] = {"pattern": kind, "ms_per_step": round(statistics.mean(tot), 4),
                              "fwd_ms": round(st["fwd"], 4), "bwd_ms": round(a_ms - st["fwd"], 4),
                              "tiles_per_bh": lay.tiles,
                              "tensor_pct_executed": tensor_pct(exec_flops(lay.tiles * Bs * Hs, d), a_ms, peaks["tf_sus"])}
            del lay
        lay = hla.HilbertLocalAttention(cfg["kind"], g, g, win, win, Bs, Hs, d, block=blk, device=dev, rpb=True)
        lay.rpb = torch.rand(lay.rpb.shape, generator=torch.Generator().manual_seed(1)) * 2 - 1
        st_fn = lambda mark, lay=lay: lay.step(q, k, v, do, mark)   # noqa: E731
        tot, _, _, _ = _timed(st_fn, vsteps, 2, flush, False, None, dist, world)
        _, st, _, _ = _timed(st_fn, vsteps, 1, flush, True, None, dist, world)
        variants["global_rpb"] = {"pattern": cfg["kind"] + " + global RPB score_mod",
                                  "ms_per_step": round(statistics.mean(tot), 4), "fwd_ms": round(st["fwd"], 4),
                                  "bwd_ms": round(st.get("bwd_pre", 0.0) + st["bwd"] + st.get("bwd_fin", 0.0), 4)}
        del lay
        if layer.hilbert and (g & (g - 1)) == 0:
            lay = hla.HilbertLocalAttention(cfg["kind"], g, g, win, win, Bs, Hs, d, block=blk, device=dev, fused=False)
            st_fn = lambda mark, lay=lay: lay.step(q, k, v, do, mark)   # noqa: E731
            tot, _, _, _ = _timed(st_fn, vsteps, 2, flush, False, None, dist, world)
            _, st, _, _ = _timed(st_fn, vsteps, 1, flush, True, None, dist, world)
            perm = {kk: round(st[kk], 4) for kk in ("perm_qkv", "perm_o", "perm_do", "perm_grads")}
            variants["unfused_reorder"] = {"pattern": cfg["kind"] + " with explicit hla_hilbert_perm passes",
                                           "ms_per_step": round(statistics.mean(tot), 4),
                                           "perm_ms": round(sum(perm.values()), 4), "perm_breakdown_ms": perm,
                                           "attn_ms": round(st["fwd"] + st.get("bwd_pre", 0.0) + st["bwd"] +
                                                            st.get("bwd_fin", 0.0), 4)}
            del lay
        rm = variants["row_major"]
        variants["speedup_attn_vs_row_major"] = round((rm["fwd_ms"] + rm["bwd_ms"]) / attn_ms, 3)
        variants["speedup_step_vs_row_major"] = round(rm["ms_per_step"] / my_ms, 3)
        variants["speedup_attn_vs_dense"] = round((variants["dense"]["fwd_ms"] + variants["dense"]["bwd_ms"]) / attn_ms, 3)
        if args.config in PAPER_SPEEDUP:
            variants["paper_speedup_fwd_bwd"] = {"value": PAPER_SPEEDUP[args.config][0],
                                                 "source": PAPER_SPEEDUP[args.config][1] + " (RTX 3080, context)"}

    # --- end to end through the public API: host -> device -> step -> host ---
    # Every step copies its inputs (Q, K, V, dO) from pinned host memory and reads its
    # results (O, dQ, dK, dV) back to pinned host memory inside the timed region.  The
    # copies run on two copy streams and the step on the compute stream, three steps in
    # flight (three layer instances = three sets of device buffers): step i+1's host->device
    # copies overlap step i's compute and step i-1's device->host copies (full-duplex link;
    # with two slots the next upload waited for the previous download, tools/probe_pcie.py).
    e2e = None
    if not args.no_e2e:
        R = 3
        hin = [x.cpu().pin_memory() for x in (q, k, v, do)]
        layers = [layer] + [hla.HilbertLocalAttention(cfg["kind"], g, g, win, win, Bs, Hs, d, block=blk, device=dev)
                            for _ in range(R - 1)]
        din = [[torch.empty_like(x) for x in (q, k, v, do)] for _ in range(R)]
        hout = [[torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in (q, q, q, q)] for _ in range(R)]
        s_in, s_out, s_cmp = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.current_stream(dev)
        ev_free = [None] * R

        def e2e_step(i):
            j = i % R
            with torch.cuda.stream(s_in):
                if ev_free[j] is not None:
                    s_in.wait_event(ev_free[j])       # slot j's buffers: step i-R fully read back
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

        esteps = max(4, args.steps)   # the pipeline fill (first upload, last download) amortised like the device loop
        for i in range(R):                          # warm-up (untimed)
            e2e_step(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_in)
        for i in range(R, R + esteps):
            e2e_step(i)
        s_out.wait_stream(s_cmp)
        e1.record(s_out)
        torch.cuda.synchronize()
        te = reduce_max_ms(e0.elapsed_time(e1) / esteps, dist if world > 1 else None, dev)
        nbytes = sum(x.numel() * x.element_size() for x in hin)
        e2e = {"value": round(te, 4), "unit": "ms", "h2d_bytes_per_step": nbytes * world,
               "d2h_bytes_per_step": nbytes * world, "steps": esteps,
               "path": "pinned host -> (copy stream) -> HilbertLocalAttention.forward/backward (compute stream) -> "
                       "(copy stream) -> pinned host; three steps in flight (triple-buffered device tensors); "
                       "per-rank shards, max over ranks; bytes = all ranks"}

    # --- roofline of the dominant kernel (share of the step) ---
    T = Bs * Hs * N                              # token-heads per launch on this rank
    kern = {
        "fwd": {"bytes": T * (8 * d + 4), "flops": 4 * 128 * 128 * d * tiles, "name": "attn_fwd_kernel"},
        "bwd": {"bytes": bwd_bytes(T, d, layer.mask, layer.fused_bwd), "flops": 10 * 128 * 128 * d * tiles,
                "name": "attn_bwd_full_kernel / attn_bwd_split_kernel"},
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
    tr = _ncu_traffic(args.config + ("@64" if blk == 64 else ""), dom)
    if tr and world == 1:
        roof["traffic"] = tr

    # --- after the timed loops: per-rank statistics over NCCL (C1, C2) ---
    ranks = gather_rank_stats([rank, b0, b1, h0, h1, my_ms, stages["fwd"], stages["bwd"], rk, rv, rbound],
                              dist if world > 1 else None, dev)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg)

    line = {
        "metric": METRIC, "value": round(step_ms, 4), "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": False,
        "scaling": "strong" if plan else "replicas", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: hla_synth splitmix64 uniform, unit variance, bf16 (no dataset)",
        "config": {"workload": "%s: %s, block %d" % (args.config, cfg["text"], blk),
                   "global_batch": B, "seq_len": N, "block": blk,
                   "parallelism": ("batch x head shards over %d ranks (plan_shards), no collective on the hot path"
                                   % world) if plan else "replicas (no batch x head partition for %d ranks)" % world,
                   "l2": "flushed between timed steps (%d MiB write, untimed); warm_l2_ms without the flush"
                         % (L2_FLUSH_BYTES >> 20),
                   "step": ("fwd+bwd (preprocess folded into the backward kernel)" if layer.fused_bwd else
                            "fwd+bwd_pre+bwd+bwd_fin") +
                           (" (Hilbert reorder fused into the kernels)" if layer.fused else ""),
                   "mask": "built once before timing: %d of %d block-%d tiles per (b,h) non-empty, %d 128 x 128 "
                           "tiles executed" % (layer.nnz, ((N + blk - 1) // blk) ** 2, blk, layer.tiles),
                   "timing": "CUDA events: one start/end pair per step (value = mean, max over ranks); "
                             "breakdown_ms = per-launch medians from a second run with one event after every "
                             "launch; " + PAPER_TIMING},
        "clocks": clocks, "e2e": e2e, "gpu_launches": layer.launches_per_step * args.steps,
        "roofline": roof, "cpu_baseline": cpu,
        "breakdown_ms": {kk: round(vv, 5) for kk, vv in stages.items()},
        "attn_ms": round(attn_ms, 4),
        "tensor_pct_executed": tensor_pct(exec_flops(tiles, d), attn_ms, peaks["tf_sus"]),
        "warm_l2_ms": round(warm_ms, 4),
        "mask_build_ms": round(statistics.median(builds), 3),
        "perm_ms": round(sum(perm.values()), 4) if perm else None,
        "ranks": [{"rank": int(r[0]), "batches": [int(r[1]), int(r[2])], "heads": [int(r[3]), int(r[4])],
                   "step_ms": round(r[5], 4), "fwd_ms": round(r[6], 4), "bwd_ms": round(r[7], 4),
                   "bwd_invariants": {"max_abs_sum_dK": r[8], "max_abs_sum_dV_minus_sum_dO": r[9],
                                      "bound": r[10], "ok": bool(r[8] <= r[10] and r[9] <= r[10])}}
                  for r in ranks],
        "paper_headlines": PAPER_HEADLINES,
        "variants": variants,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args, argv))
    if args.impl == "reference":
        if args.config in STACK:
            if dist_env()[0] == 0:
                print(json.dumps({"impl": "reference", "unavailable": "the oracle leg covers cfg1-cfg4 only"}))
            return
        run_reference(args, CONFIGS[args.config])
        return
    if args.config in STACK:
        run_stack(args)
    else:
        run_single(args)


if __name__ == "__main__":
    main()
