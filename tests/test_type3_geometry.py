"""Type-3 grid geometry on the host (reference
transforms.py:233-264, tests/test_transforms.py type3_geometry_*): the
frozen example, degenerate targets and the two design inequalities
(X / gamma <= pi (1 - w / n), gamma S <= n / (2 sigma)) on random clouds,
plus the recentring rule.  Host-side arithmetic only (no GPU)."""
import numpy as np
import pytest

from paper_1808_06736_b200.grid import next_smooth
from paper_1808_06736_b200.kernel import params_for_width
from paper_1808_06736_b200.transforms import _axis_shift, plan_type3_geometry


def test_geometry_frozen_example():
    p = params_for_width(7, 2.0)
    geo = plan_type3_geometry([np.array([-np.pi, np.pi])], [np.array([-50.0, 50.0])], p, 2.0)
    # n = next_smooth(ceil((2 sigma / pi) X S) + w) = next_smooth(200 + 7)
    assert geo.sizes == (next_smooth(207),) == (216,)
    assert geo.x_shift == (0.0,) and geo.s_shift == (0.0,)
    assert geo.gamma[0] == pytest.approx(216 / (4.0 * 50.0), rel=1e-15)


def test_geometry_degenerate_targets():
    # one target: S = 0 -> half-width 1 in the size rule, the smallest grid
    p = params_for_width(7, 2.0)
    geo = plan_type3_geometry([np.array([0.3])], [np.array([5.0])], p, 2.0)
    assert geo.sizes == (next_smooth(2 * p.w),)
    assert geo.s_half_width == (0.0,)


@pytest.mark.parametrize("sigma", [2.0, 1.25])
def test_geometry_inequalities_random(sigma):
    rng = np.random.default_rng(8)
    p = params_for_width(7, sigma)
    for _ in range(40):
        x = rng.uniform(-rng.uniform(0.1, 3), rng.uniform(0.1, 3), 20)
        s = rng.uniform(-rng.uniform(1, 300), rng.uniform(1, 300), 20)
        geo = plan_type3_geometry([x], [s], p, sigma)
        n, X, S, g = geo.sizes[0], geo.x_half_width[0], geo.s_half_width[0], geo.gamma[0]
        assert X / g <= np.pi * (1.0 - p.w / n) * (1 + 1e-12)
        assert g * S <= n / (2.0 * sigma) * (1 + 1e-12)
        # the shifts recentre: half-widths never exceed the raw extents
        assert X <= np.abs(x).max() * (1 + 1e-15) and S <= np.abs(s).max() * (1 + 1e-15)


def test_axis_shift_rule():
    assert _axis_shift(10.0, 10.2) == pytest.approx(10.1)
    assert _axis_shift(-5.0, 5.0) == 0.0
    assert _axis_shift(-1.0, 3.0) == 0.0  # halves the range by less than 2x: kept
    assert _axis_shift(2.0, 3.0) == pytest.approx(2.5)
