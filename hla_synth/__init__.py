"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no permutation, mask or
attention); it only turns (seed, tensor_id, linear index) into numbers, so that
the oracle and the CUDA path see identical bf16 values:

  u = splitmix64(seed ^ (tensor_id << 56) ^ idx) >> 40          (24 bits)
  x = (u * 2^-24 * 2 - 1) * sqrt(3)   in fp32  (uniform, unit variance)
  bf16 = round-to-nearest-even of the fp32 bits

idx is the linear index in the [B, N, heads, d] tensor in GRID (row-major cell)
order.  tensor_id: Q=1, K=2, V=3, dO=4.  A "sharp" variant multiplies Q by 4.

Two implementations of the same counter-based generator are provided: numpy
(uint64) and torch (int64 with masked logical shifts; runs on CPU or CUDA).
Tests check that they agree bit for bit.
"""

import math

import numpy as np

TENSOR_ID = {"q": 1, "k": 2, "v": 3, "do": 4}

_GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB


def splitmix64_np(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(_GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
        return z ^ (z >> np.uint64(31))


def _bf16_rne_bits(f32):
    bits = f32.view(np.uint32).astype(np.uint64)
    rounded = (bits + np.uint64(0x7FFF) + ((bits >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return rounded.astype(np.uint16)


def bf16_bits_to_f32(bits16):
    return (np.asarray(bits16, dtype=np.uint32) << np.uint32(16)).view(np.float32)


def uniform_np(shape, seed, tensor_id, scale=1.0):
    """fp32 numpy array of bf16-representable values (the exact values both sides use)."""
    n = int(np.prod(shape))
    idx = np.arange(n, dtype=np.uint64)
    key = np.uint64((seed ^ (tensor_id << 56)) & 0xFFFFFFFFFFFFFFFF)
    u = splitmix64_np(key ^ idx) >> np.uint64(40)
    x = ((u.astype(np.float32) * np.float32(2.0 ** -24) * np.float32(2.0) - np.float32(1.0))
         * np.float32(math.sqrt(3.0)))
    x = (x * np.float32(scale)).astype(np.float32)
    return bf16_bits_to_f32(_bf16_rne_bits(x)).reshape(shape)


# --------------------------------------------------------------------------- torch
def _to_signed(v):
    return v - (1 << 64) if v >= (1 << 63) else v


def _lsr(z, k):
    """Logical right shift of int64 (two's complement) tensor."""
    import torch  # noqa: F401
    return (z >> k) & ((1 << (64 - k)) - 1)


def splitmix64_torch(x):
    z = x + _to_signed(_GOLDEN)
    z = (z ^ _lsr(z, 30)) * _to_signed(_M1)
    z = (z ^ _lsr(z, 27)) * _to_signed(_M2)
    return z ^ _lsr(z, 31)


def uniform_torch(shape, seed, tensor_id, scale=1.0, device="cpu", chunk=1 << 26):
    """bf16 torch tensor with the same values as uniform_np (generated on `device`)."""
    import torch
    n = int(np.prod(shape))
    out = torch.empty(n, dtype=torch.bfloat16, device=device)
    key = _to_signed((seed ^ (tensor_id << 56)) & 0xFFFFFFFFFFFFFFFF)
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        idx = torch.arange(c0, c1, dtype=torch.int64, device=device)
        u = _lsr(splitmix64_torch(idx ^ key), 40)
        x = (u.to(torch.float32) * (2.0 ** -24) * 2.0 - 1.0) * math.sqrt(3.0)
        x = x * scale
        out[c0:c1] = x.to(torch.bfloat16)          # torch's bf16 cast is RNE
    return out.view(*shape)


def uniform_torch_block(shape, b0, b1, h0, h1, seed, tensor_id, scale=1.0, device="cpu"):
    """The [b0:b1, :, h0:h1, :] block of uniform_torch(shape, ...) for shape = (B, N, H, d),
    generated from its GLOBAL linear indices (a rank's shard holds exactly the values of the
    global tensor -- multi-GPU shards, bench.py plan_shards)."""
    import torch
    B, N, H, d = shape
    out = torch.empty((b1 - b0, N, h1 - h0, d), dtype=torch.bfloat16, device=device)
    key = _to_signed((seed ^ (tensor_id << 56)) & 0xFFFFFFFFFFFFFFFF)
    hd = torch.arange(h0, h1, dtype=torch.int64, device=device)[:, None] * d + torch.arange(d, device=device)[None, :]
    rows = max(1, (1 << 24) // max(1, (h1 - h0) * d))
    for b in range(b0, b1):
        for n0 in range(0, N, rows):
            n1 = min(N, n0 + rows)
            tok = (b * N + torch.arange(n0, n1, dtype=torch.int64, device=device)) * (H * d)
            idx = tok[:, None, None] + hd[None, :, :]
            u = _lsr(splitmix64_torch(idx ^ key), 40)
            x = (u.to(torch.float32) * (2.0 ** -24) * 2.0 - 1.0) * math.sqrt(3.0)
            out[b - b0, n0:n1] = (x * scale).to(torch.bfloat16)
    return out


def attention_inputs_block(B, N, H, d, b0, b1, h0, h1, seed=0, sharp=False, device="cpu"):
    """q, k, v, dO restricted to batches [b0, b1) and heads [h0, h1) of the global tensors."""
    qscale = 4.0 if sharp else 1.0
    shape = (B, N, H, d)
    return tuple(uniform_torch_block(shape, b0, b1, h0, h1, seed, t, sc, device)
                 for t, sc in ((1, qscale), (2, 1.0), (3, 1.0), (4, 1.0)))


def attention_inputs(B, N, H, d, seed=0, sharp=False, backend="torch", device="cpu"):
    """q, k, v, dO in grid order, layout [B, N, heads, d]."""
    qscale = 4.0 if sharp else 1.0
    shape = (B, N, H, d)
    if backend == "numpy":
        return (uniform_np(shape, seed, 1, qscale), uniform_np(shape, seed, 2),
                uniform_np(shape, seed, 3), uniform_np(shape, seed, 4))
    return (uniform_torch(shape, seed, 1, qscale, device), uniform_torch(shape, seed, 2, 1.0, device),
            uniform_torch(shape, seed, 3, 1.0, device), uniform_torch(shape, seed, 4, 1.0, device))
