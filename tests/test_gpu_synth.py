"""The device generator (k_synth.cu) draws exactly the host generator's bits (inputs/synth_host.cpp):
indices and values of a 1e6-draw slice of configs 3 and 4, so the oracle (host inputs) and the GPU
path (device inputs) see the same observations at any size."""
import numpy as np
import pytest

from inputs import configs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("which", ["config3", "config4"])
def test_device_generator_matches_host(ctx, which):
    import paper_2603_25691_b200 as cp
    c = getattr(configs, which)()
    q = 1_000_000
    idx_d, vals_d = cp.synth_observations_device(c, ctx, q)
    idx_h, vals_h = configs.generate_host(c, 0, q)
    assert np.array_equal(idx_d.cpu().numpy(), idx_h)
    assert np.array_equal(vals_d.cpu().numpy().view(np.uint64), vals_h.view(np.uint64))
