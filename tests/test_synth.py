"""The shared input generator: seeded, position-stable (independent of sharding), unit rows, bf16 RNE."""
import numpy as np
import torch

from synth import make_features, shard


def test_rows_position_stable():
    I, T = make_features(10000, 32, seed=3)
    I2, T2 = make_features(10000, 32, seed=3, row0=4000, rows=5000)
    assert torch.equal(I[4000:9000], I2) and torch.equal(T[4000:9000], T2)


def test_unit_norm_and_rounding():
    I, T = make_features(512, 64, seed=1, dtype=torch.float32)
    assert np.allclose(I.norm(dim=1).numpy(), 1.0, atol=1e-6)
    Ib, _ = make_features(512, 64, seed=1)
    assert torch.equal(Ib, I.to(torch.bfloat16))


def test_paired_correlated_and_shard():
    I, T = make_features(2048, 128, seed=0, dist="paired")
    cos = (I.float() * T.float()).sum(1).mean().item()
    assert 0.6 < cos < 0.8
    parts = [shard(I, r, 4) for r in range(4)]
    assert torch.equal(torch.cat(parts), I)


def test_onehot_device_matches_host():
    from synth import make_onehot_device
    I, T = make_features(300, 16, dist="onehot", K=8)
    Id, Td = make_onehot_device(300, 16, 8, "cpu")
    assert torch.equal(I, Id) and torch.equal(T, Td)
