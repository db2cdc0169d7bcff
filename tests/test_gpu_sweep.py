"""sweep_conv on the B200 (kernel-level conv passes, CUDA-event timed)."""

import pytest

from paper_1909_12291_b200 import sweep

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_sweep_conv_small_grid(precision):
    grid = sweep.SweepGrid(in_channels=(3, 16), out_channels=(8, 12), kernels=(1, 3, 9), strides=(1, 2),
                           batch_sizes=(8,), height=8, width=8)
    rows, skipped = sweep.sweep_conv(grid, reps=3, precision=precision, inner=2)
    assert len(rows) + len(skipped) == grid.size()
    assert len(skipped) == 2 * 2 * 2  # kernel 9 > 8x8 input, every (cin, cout, stride)
    assert all(r.median_forward_backward_s > 0 and r.flops_per_s > 0 for r in rows)
    prior = sweep.build_prior(rows, k=4)
    assert abs(sum(prior.kernel.values()) - 1.0) < 1e-12
    with pytest.raises(ValueError):
        sweep.sweep_conv(grid, reps=2)
