"""The shared input generator: numpy and torch implementations agree bit for bit,
values are bf16-representable with the intended distribution."""

import numpy as np
import torch

import hla_synth


def test_splitmix_known_values():
    # splitmix64 reference outputs for seed state 0 -> first outputs of the
    # published generator (x += golden; mix) with x = 0, 1, 2.
    out = hla_synth.splitmix64_np(np.array([0, 1, 2], dtype=np.uint64))
    assert int(out[0]) == 0xE220A8397B1DCDAF
    assert int(out[1]) == 0x910A2DEC89025CC1
    t = hla_synth.splitmix64_torch(torch.tensor([0, 1, 2], dtype=torch.int64))
    assert [v & 0xFFFFFFFFFFFFFFFF for v in t.tolist()] == [int(x) for x in out]


def test_numpy_torch_agree():
    shape = (2, 64, 3, 32)
    for tid, sc in ((1, 1.0), (2, 1.0), (1, 4.0), (4, 1.0)):
        a = hla_synth.uniform_np(shape, 7, tid, sc)
        b = hla_synth.uniform_torch(shape, 7, tid, sc).float().numpy()
        assert np.array_equal(a, b)


def test_distribution():
    x = hla_synth.uniform_np((1 << 16,), 0, 1)
    assert abs(x.mean()) < 0.02 and abs(x.var() - 1.0) < 0.02
    assert np.abs(x).max() <= np.sqrt(3) + 1e-2
    bits = x.view(np.uint32)
    assert not (bits & 0xFFFF).any()          # exactly bf16-representable


def test_block_generator_matches_global_tensor():
    """A multi-GPU shard ([b0:b1, :, h0:h1]) holds exactly the global tensor's values."""
    import torch
    full = hla_synth.attention_inputs(3, 16, 4, 8, seed=5, sharp=True)
    for b0, b1, h0, h1 in ((0, 3, 0, 4), (1, 3, 1, 3), (2, 3, 0, 1)):
        blk = hla_synth.attention_inputs_block(3, 16, 4, 8, b0, b1, h0, h1, seed=5, sharp=True)
        assert all(torch.equal(f[b0:b1, :, h0:h1], b) for f, b in zip(full, blk))
