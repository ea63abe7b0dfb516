"""The seeded input library (inputs/): host side of the counter-based generator of configs 3/4
and its deterministic transcendental pieces (no product library involved)."""
import math

import numpy as np

import inputs
from inputs import configs


def test_log_cos_accuracy():
    L = inputs.lib()
    xs = np.concatenate([np.geomspace(2.0 ** -53, 1.0, 2000), np.linspace(0.5, 1.0, 2000)])
    for x in xs:
        ref = math.log(x)
        assert abs(L.inp_syn_log(float(x)) - ref) <= 4e-16 * max(1.0, abs(ref))
    for f in np.linspace(0.0, 1.0, 4001)[:-1]:
        assert abs(L.inp_syn_cos2pi(float(f)) - math.cos(2 * math.pi * f)) <= 1e-15


def test_counter_based_slices_and_threads():
    c = configs.config4()
    i_all, v_all = configs.generate_host(c, 0, 5000, threads=1)
    i_par, v_par = configs.generate_host(c, 0, 5000, threads=4)
    assert np.array_equal(i_all, i_par) and np.array_equal(v_all.view(np.uint64), v_par.view(np.uint64))
    i_mid, v_mid = configs.generate_host(c, 1234, 4321, threads=3)   # any slice of the counter space
    assert np.array_equal(i_mid, i_all[:, 1234:4321])
    assert np.array_equal(v_mid.view(np.uint64), v_all[1234:4321].view(np.uint64))
    i_nov, v_none = configs.generate_host(c, 0, 5000, values=False)
    assert v_none is None and np.array_equal(i_nov, i_all)


def test_config4_distribution():
    c = configs.config4()
    idx, vals = configs.generate_host(c, 0, 400_000)
    for m, n in enumerate(c.shape):
        assert idx[m].min() >= 0 and idx[m].max() < n
    head = np.mean(idx[0] == 0)
    assert abs(head - 0.1605) < 0.005, head                  # P(i_1 = 0) = 16.05 %
    assert abs(np.mean(idx[0] < 10) - 0.43) < 0.01           # top 10: 43 %
    for m in (1, 2):                                         # uniform modes
        assert abs(idx[m].mean() - (c.shape[m] - 1) / 2) < 3.0
    # values = model + N(0, 0.1^2): residual against the rank-64 model
    model = np.ones((idx.shape[1], c.r))
    for m in range(3):
        model *= c.factors[m][idx[m]]
    res = vals - model.sum(axis=1)
    assert abs(res.mean()) < 2e-3 and abs(res.std() - 0.1) < 2e-3


def test_config3_uniform():
    c = configs.config3()
    idx, vals = configs.generate_host(c, 10_000_000, 10_100_000)
    assert idx.shape == (4, 100_000) and np.isfinite(vals).all()
    for m, n in enumerate(c.shape):
        assert idx[m].min() >= 0 and idx[m].max() < n
        assert abs(idx[m].mean() - (n - 1) / 2) < 0.02 * n
