"""The §5 timing model: fit recovers known parameters; limits."""
import numpy as np
import pytest

from paper_1703_00186_b200 import perfmodel as pm


def test_fit_recovers_parameters():
    true = pm.Params(alpha=9e-11, beta=2e-8, gamma=2.3e-9, delta=5e-9)
    rng = np.random.default_rng(0)
    samples = []
    for lx in (256, 512, 1024, 2048):
        for ly in (1024, 2048, 4096, 8192):
            t = true.alpha * lx * ly + true.beta * lx
            samples.append((lx, ly, t * (1 + 1e-6 * rng.standard_normal())))
    a, b = pm.fit_bulk(samples)
    assert a == pytest.approx(true.alpha, rel=1e-4)
    assert b == pytest.approx(true.beta, rel=1e-2)
    d = pm.fit_rows([(ly, true.delta * ly) for ly in (1024, 4096, 8192)])
    assert d == pytest.approx(true.delta, rel=1e-12)


def test_model_limits():
    p = pm.Params(alpha=1e-10, beta=0.0, gamma=0.0, delta=0.0)
    assert pm.speedup(p, 8192, 8192, 1) == pytest.approx(1.0)
    for n in (2, 4, 8):
        assert pm.speedup(p, 8192, 8192, n) == pytest.approx(n)       # perfect strong scaling
        assert pm.weak_efficiency(p, 4096, 8192, n) == pytest.approx(1.0)
    # communication-bound regime: T -> gamma Ly + delta Ly, S_r saturates
    q = pm.Params(alpha=1e-10, beta=0.0, gamma=1e-5, delta=0.0)
    assert pm.step_time(q, 1080, 5736, 36) == pytest.approx(1e-5 * 5736)
    assert pm.speedup(q, 1080, 5736, 36) < 36


def test_paper_shape_crossover():
    """T ~ T_a while alpha (Lx/n) Ly + beta Lx/n > gamma Ly, T ~ T_b beyond."""
    p = pm.Params(alpha=1e-10, beta=0.0, gamma=1e-10 * 1080 / 24.5, delta=1e-9)
    n_cross = next(n for n in range(1, 100) if p.gamma * 5736 > p.alpha * (1080 / n) * 5736)
    assert 20 <= n_cross <= 30
