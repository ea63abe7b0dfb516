"""A/B timings of the solver-level paths (one process, env toggles read per call):
  config 1 PCG solve: host loop (CPHIFI_PCG_GRAPH=0) vs device-resident CUDA-graph loop
  aligned configs 0 / 2: MTTKRP v1 vs v2, decoupled solve via 4 DMMA GEMMs vs the 2-launch sandwich
  python profiles/prof_solves.py [--large 1]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench_secondary as bs  # noqa: E402
import paper_2603_25691_b200 as cp  # noqa: E402
from inputs import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--large", type=int, default=0)
    args = ap.parse_args()
    ctx = cp.Context(0)
    c = configs.config1()
    n, r = c.shape[0], c.r
    mode = cp.RkhsMode(c.points, c.ell, c.lam, ctx=ctx)
    p = cp.make_unaligned_subproblem(cp.ObservationSet(c.shape, c.idx, c.vals),
                                     cp.KruskalModel([np.zeros((n, r))] + c.factors[1:]), 0, mode, c.rho)
    ws, hs = {}, {}
    for g in ("0", "1"):
        os.environ["CPHIFI_PCG_GRAPH"] = g
        walls = []
        for _ in range(6):
            rep = cp.SolveReport()
            w = cp.solve_unaligned_pcg(p, cp.PcgConfig(c.tol, c.max_iter, record_history=True), rep)
            walls.append(rep.wall_time_s)
        ws[g] = w
        hs[g] = list(rep.residual_history)
        print(f"config1 PCG graph={g}: iters {rep.iterations} rel {rep.relative_residual:.3e} "
              f"wall first {walls[0]*1e3:.3f} ms, median rest {np.median(walls[1:])*1e3:.3f} ms, "
              f"setup {rep.setup_s*1e3:.3f} ms hist {len(rep.residual_history)}")
    print("graph vs host W rel diff", np.linalg.norm(ws["0"] - ws["1"]) / np.linalg.norm(ws["0"]),
          "hist equal", hs["0"] == hs["1"])
    os.environ.pop("CPHIFI_PCG_GRAPH")
    fp = bs.fp64_peaks(ctx)["dmma_tflops"]
    for which in ("config0", "config2"):
        for v1, v3, sw in (("1", "0", "0"), ("0", "0", "1"), ("0", "1", "0"), ("0", "1", "1")):
            os.environ["CPHIFI_MTTKRP_V1"] = v1
            os.environ["CPHIFI_MTTKRP_V3"] = v3
            os.environ["CPHIFI_SANDWICH"] = sw
            t0 = time.perf_counter()
            o = bs.aligned(which, ctx, 20, fp)
            print(f"{which} mttkrp_v1={v1} v3={v3} sandwich={sw}: solve {o['solve_ms']*1e3:.1f} us "
                  f"(mttkrp {o['mttkrp_ms']*1e3:.1f}, gram {o['gram_ms']*1e3:.1f}, decoupled {o['decoupled_ms']*1e3:.1f}) "
                  f"roofline {o['roofline_frac']:.3f}  [{time.perf_counter()-t0:.1f}s]")
    for k in ("CPHIFI_MTTKRP_V1", "CPHIFI_MTTKRP_V3", "CPHIFI_SANDWICH"):
        os.environ.pop(k)


if __name__ == "__main__":
    main()
