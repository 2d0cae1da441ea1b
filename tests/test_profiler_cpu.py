"""NEXT-1 pipeline profiler host logic, pinned by SPEC.md's worked example."""
import pytest

from paper_2504_09345_b200 import profiler


def test_spec_example_n_real_700():
    # slope 2e-4 s/token, intercept 0.01 s, per-layer IO 0.15 s -> n_real = 700
    ns = [100, 200, 400, 800]
    ts = [0.01 + 2e-4 * n for n in ns]
    slope, icpt = profiler.fit_line(ns, ts)
    assert slope == pytest.approx(2e-4) and icpt == pytest.approx(0.01)
    assert profiler.n_real(slope, icpt, 0.15) == pytest.approx(700)


def test_fit_line_least_squares_noise():
    ns = [1, 2, 3, 4]
    ts = [2.1, 3.9, 6.1, 7.9]          # y = 2x + 0 with +-0.1 noise
    s, b = profiler.fit_line(ns, ts)
    assert s == pytest.approx(1.96) and b == pytest.approx(0.1)


def test_fit_line_rejects_degenerate():
    with pytest.raises(ValueError):
        profiler.fit_line([5], [1.0])
    with pytest.raises(ValueError):
        profiler.fit_line([5, 5], [1.0, 2.0])
    with pytest.raises(ValueError):
        profiler.n_real(0.0, 1.0, 2.0)
