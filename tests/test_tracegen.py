"""The seeded input generator (holds none of the method's arithmetic): deterministic,
shard/chunk-consistent, and shaped like the configured workloads."""
import numpy as np

from paper_2410_12588_b200 import tracegen as tg


def test_counter_generator_is_window_consistent():
    spec = tg.make_spec(tg.CONFIGS["C3"], n_series=64, T=5000)
    full = tg.generate(spec, 0, 64, 0, 3000)
    part = tg.generate(spec, 10, 20, 1000, 1500)
    np.testing.assert_array_equal(part, full[10:30, 1000:2500])


def test_normals_are_standard():
    z = tg.std_normal(7, np.arange(1000, dtype=np.uint64)[:, None], np.arange(200, dtype=np.uint64)[None, :])
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01


def test_c1_shape():
    spec = tg.make_spec(tg.CONFIGS["C1"], sigma=0.0)
    x = tg.generate(spec)
    assert x.shape == (1, 1000)
    np.testing.assert_allclose(x[0, :600], 1.0)
    np.testing.assert_allclose(x[0, 600:], 1.5)


def test_c2_episodes_are_synchronous():
    spec = tg.make_spec(tg.CONFIGS["C2"], n_series=8, T=10000)
    eps = [spec.episodes(s) for s in range(8)]
    assert all(e == eps[0] for e in eps) and len(eps[0]) == 6
    for a, b, sev in eps[0]:
        assert 0 <= a < b <= 10000 and 1.15 <= sev <= 1.25


def test_c3_episode_statistics():
    spec = tg.make_spec(tg.CONFIGS["C3"], n_series=20000, T=100000)
    n = np.diff(spec.ep_off)
    frac = (n > 0).mean()
    assert 0.37 < frac < 0.43
    sev = np.exp(spec.ep_logsev)
    assert sev.min() >= 1.39 and sev.max() <= 6.7
    dur = spec.ep_end - spec.ep_start
    assert dur.max() <= 20571 and dur.min() >= 1
