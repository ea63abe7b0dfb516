"""Full-size PCG parity for BASELINE configs 3 and 4 (q = 2e8 / 1e9 draws) against fixtures the
ORACLE computed on the CPU (tests/golden/make_pcg_fixtures.py: the streaming restatement of
observations.hpp:174-198 inside the reference PCG, solvers.hpp:38-88 / unaligned.hpp:143-161, on
the same seeded draws — the host generator is bit-identical to the device one,
tests/test_gpu_synth.py — with the same kernel matrix K).  No GPU time is spent on the oracle.

Asserted (north_star): iterations within +-1 and the final relative residual <= tol; also the
residual histories over the common prefix, the right-hand side B, the true residual of the device
W under the REFERENCE operator (K itself, not the clamped eigen-reconstruction the device PCG
iterates with), and A = K W (als.hpp:214), the quantity the ALS consumes.  eig(K) is not shared:
the device uses cuSOLVER's, the oracle LAPACK's, one more reason W itself is compared
only through K W (the ill-conditioned directions of W are set by rho and the eigensolver)."""
import os

import numpy as np
import pytest

from inputs import configs
from oracle import oracle as orc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.fixture(scope="module")
def solved(ctx):
    """Device solves of configs 3 and 4 (both operator forms), cached for the module."""
    import torch

    import paper_2603_25691_b200 as cp
    out = {}
    for which in ("config3", "config4"):
        fx = np.load(os.path.join(GOLD, f"{which}_pcg.npz"))
        cfg = getattr(configs, which)()
        n, r = cfg.shape[0], cfg.r
        kern = orc.matern32_kernel(cfg.points, cfg.ell) if cfg.kernel == "matern32" else \
            orc.gaussian_kernel(cfg.points, cfg.ell)
        idx, vals = cp.synth_observations_device(cfg, ctx)
        chk = [int(v) for v in idx.to(torch.int64).sum(dim=1).cpu().numpy()]
        mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel_matrix=kern)
        obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), cfg.q, keepalive=(idx, vals),
                                    coalesce=cfg.coalesce)
        p = cp.make_unaligned_subproblem(obs, cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:]), 0, mode,
                                         cfg.rho)
        del idx, vals
        obs.release_inputs()
        torch.cuda.empty_cache()
        res = {"fx": fx, "kern": kern, "chk": chk, "b": p.b, "default_op": p.operator()}
        for op in ("gram", "stream"):
            p.set_operator(op)
            rep = cp.SolveReport()
            w = cp.solve_unaligned_pcg(p, cp.PcgConfig(cfg.tol, cfg.max_iter, record_history=True), rep)
            # true residual under the reference operator (original K, unaligned.hpp:101-115), evaluated
            # by the device operator in the original basis
            rhs = (kern @ res["b"]).reshape(-1, order="F")
            aw = cp.unaligned_matvec(p, w.reshape(-1, order="F"))
            res[op] = {"w": w, "it": rep.iterations, "rel": rep.relative_residual,
                       "hist": np.array(rep.residual_history),
                       "true_rel": float(np.linalg.norm(rhs - aw) / np.linalg.norm(rhs))}
        out[which] = res
        del p, obs, mode
        torch.cuda.empty_cache()
    return out


@pytest.mark.parametrize("which", ["config3", "config4"])
@pytest.mark.parametrize("op", ["gram", "stream"])
def test_full_size_pcg_vs_oracle_fixture(solved, which, op):
    res = solved[which]
    fx, kern = res["fx"], res["kern"]
    cfg = getattr(configs, which)()
    d = res[op]
    assert res["chk"] == [int(v) for v in fx["idx_checksum"]]  # the same draws as the oracle's
    assert rel(res["b"], fx["b"]) < 1e-12                          # B = sampled_mttkrp(values)
    assert abs(d["it"] - int(fx["iterations"])) <= 1, (d["it"], int(fx["iterations"]))
    assert d["rel"] <= cfg.tol
    assert d["true_rel"] <= 10 * cfg.tol, d["true_rel"]
    h, ho = d["hist"], fx["history"]
    m = min(len(h), len(ho))
    hist_rel = float(np.max(np.abs(h[:m] - ho[:m]) / ho[:m]))
    kw_rel = rel(kern @ d["w"], fx["a"])
    print(f"{which} {op}: iterations {d['it']} (oracle {int(fx['iterations'])}), rel {d['rel']:.3e}, "
          f"true rel {d['true_rel']:.3e}, history max rel diff {hist_rel:.3e}, |KW - KW_orc| {kw_rel:.3e}, "
          f"|W - W_orc| {rel(d['w'], fx['w']):.3e}")
    # measured (B200, this fixture): history 1.6e-7 (config 3, 5 iterations) and 4.6e-4 (config 4,
    # 75 iterations of an ill-conditioned CG, different eigenbases); K W 2.5e-8 / 2.8e-8 while W
    # itself differs by 1.5 % / 97 % (its components along K's null space are set by rho alone)
    assert hist_rel <= 1e-3
    assert kw_rel <= 1e-6


def test_drop_in_default_is_row_gram(solved):
    """The drop-in default at configs 3 / 4 is the row-Gram operator (AUTO at plan creation)."""
    assert solved["config3"]["default_op"] == "gram" and solved["config4"]["default_op"] == "gram"
