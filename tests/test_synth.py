"""The shared input generator: determinism, shard independence, distribution sanity."""
import torch

from synth import kv_cache_iid, normal_f64, q_iid, splitmix64, structured_qkv


def test_splitmix_reference_values():
    # SplitMix64 outputs for state 0 (seed 0): first three values of the reference generator
    # (Steele/Lea/Flood, "Fast splittable PRNGs"; state advanced by the golden gamma).
    want = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    g = 0x9E3779B97F4A7C15
    wrap = lambda x: x - (1 << 64) if x >= (1 << 63) else x
    st = torch.tensor([wrap((i * g) & 0xFFFFFFFFFFFFFFFF) for i in range(3)], dtype=torch.int64)
    out = splitmix64(st)
    assert [int(x) & 0xFFFFFFFFFFFFFFFF for x in out] == want


def test_deterministic_and_shardable():
    a = q_iid(7, 13, 0, 4, 64, 32)
    b = q_iid(7, 13, 2, 2, 64, 32)           # heads 2, 3 generated alone
    assert torch.equal(a[2:], b)
    assert torch.equal(a, q_iid(7, 13, 0, 4, 64, 32))
    assert not torch.equal(a, q_iid(8, 13, 0, 4, 64, 32))
    assert not torch.equal(a, q_iid(7, 12, 0, 4, 64, 32))


def test_capacity_zero_padded():
    k, v = kv_cache_iid(0, 0, 2, 85, 16, capacity=96)
    assert k.shape == (2, 96, 16) and (k[:, 85:] == 0).all() and (v[:, 85:] == 0).all()


def test_normal_moments():
    z = normal_f64(0, 1, 0, 200000)
    assert abs(z.mean().item()) < 0.01 and abs(z.std().item() - 1) < 0.01


def test_structured_shapes():
    q, k, v = structured_qkv(0, [1, 2, 4, 6, 8, 12], 6, 6, 0, 2, 16)
    assert q.shape == (2, 144, 16) and k.shape == (2, 265, 16) and v.dtype == torch.bfloat16
