"""Launch list of ONE warm PCG solve (row-Gram operator) at full size, for the per-iteration
kernel breakdown.  The first solve captures the device-loop graph; the second runs between
cudaProfilerStart/Stop so that

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/pcg4.csv python profiles/prof_pcg_launches.py --config 4

lists exactly that solve's kernels (run through the host-driven loop, CPHIFI_PCG_GRAPH=0: the
same kernels as the graph's WHILE body, which ncu does not replay) (without ncu it prints the solve's wall time).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_25691_b200 as cp  # noqa: E402
from inputs import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--ab", type=int, default=0, help="time N graph solves then N host-loop solves (no profiler range)")
    args = ap.parse_args()
    ctx = cp.Context(0)
    cfg = getattr(configs, f"config{args.config}")()
    n, r, q = cfg.shape[0], cfg.r, cfg.q
    idx, vals = cp.synth_observations_device(cfg, ctx)
    torch.cuda.synchronize()
    mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
    obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), q, keepalive=(idx, vals),
                                coalesce=cfg.coalesce)
    p = cp.make_unaligned_subproblem(obs, cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:]), 0, mode, cfg.rho)
    del idx, vals
    obs.release_inputs()
    torch.cuda.empty_cache()
    p.set_operator("gram")
    mode.eig()
    if args.ab:
        for mode_g in ("1", "0"):
            os.environ["CPHIFI_PCG_GRAPH"] = mode_g
            for _ in range(args.ab):
                rep = cp.SolveReport()
                cp.solve_unaligned_pcg(p, cp.PcgConfig(cfg.tol, cfg.max_iter), rep)
                print(f"graph={mode_g}: iterations {rep.iterations} wall {rep.wall_time_s * 1e3:.3f} ms setup {rep.setup_s * 1e3:.3f} ms",
                      flush=True)
        return
    for rep_i in range(3):
        rep = cp.SolveReport()
        if rep_i == 2:
            os.environ["CPHIFI_PCG_GRAPH"] = "0"  # host loop: ncu does not replay conditional graph nodes
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
        cp.solve_unaligned_pcg(p, cp.PcgConfig(cfg.tol, cfg.max_iter), rep)
        if rep_i == 2:
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
        print(f"solve {rep_i}: iterations {rep.iterations} rel {rep.relative_residual:.3e} wall {rep.wall_time_s * 1e3:.3f} ms",
              flush=True)


if __name__ == "__main__":
    main()
