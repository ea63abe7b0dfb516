# host-buffer matvec: pinned large x / y by DMA around an operator-only graph; e2e at config 4
python -m pytest tests/test_gpu_paths.py -x -q > gpurun_out/dma_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/dma_tests.log
python bench.py --steps 30 --warmup 3 --secondary 0 --cpu-seconds 1 > gpurun_out/bench_dma.json 2>&1; echo "bench rc=$?"
CPHIFI_SOLVE_TIMING=1 python -c "
import sys; sys.argv=['x']
import bench_secondary as bs, paper_2603_25691_b200 as cp, numpy as np
from inputs import configs
cfg = configs.config4(); ctx = cp.Context(0); n, r = cfg.shape[0], cfg.r
idx, vals = cp.synth_observations_device(cfg, ctx)
mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), cfg.q, keepalive=(idx, vals), coalesce=cfg.coalesce)
p = cp.make_unaligned_subproblem(obs, cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:]), 0, mode, cfg.rho)
p.set_operator('stream'); p.qpass_plan()
print(bs.config4_solves(cp, p, obs, mode, cfg))
" > gpurun_out/stream_setup.log 2>&1
