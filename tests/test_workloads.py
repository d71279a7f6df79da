"""The C4 / C5 per-shard generator (workloads.noisy_lowrank_shard) is shard-count independent: the
rows a rank generates for itself equal the same rows of a one-shard generation, so a
row-sharded run at any world size factorises the same global X."""
import numpy as np
import pytest

from paper_1711_02037_b200 import workloads


@pytest.mark.parametrize("world", [2, 3, 8])
def test_shards_concatenate_to_whole(world):
    m, n, r = 9000, 300, 7
    whole = workloads.noisy_lowrank_shard(5, m, n, r, 0.5, 0.1, 0, m, device="cpu", block=1024).numpy()
    parts = []
    for rank in range(world):
        lo, hi = m * rank // world, m * (rank + 1) // world
        parts.append(workloads.noisy_lowrank_shard(5, m, n, r, 0.5, 0.1, lo, hi - lo, device="cpu", block=1024).numpy())
    np.testing.assert_array_equal(np.concatenate(parts), whole)


def test_distribution_matches_config_wording():
    m, n, r, s = 4096, 2000, 40, 0.5
    x = workloads.noisy_lowrank_shard(0, m, n, r, s, 0.1, 0, m, device="cpu").numpy().astype(np.float64)
    assert (x >= 0).all()
    mean_lr = workloads.lowrank_expected_mean(r, s)
    # the low-rank part's mean is rank (1-s)^2 2/pi; |N(0, 0.1 mean)| adds 0.1 mean sqrt(2/pi)
    expect = mean_lr * (1 + 0.1 * np.sqrt(2 / np.pi))
    assert abs(x.mean() / expect - 1) < 0.05
