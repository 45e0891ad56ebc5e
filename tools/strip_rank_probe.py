"""One rank's share of an N-GPU C5 strip run, measured on one GPU under
torchrun (world 1, NCCL): the device time per iteration and the host time the
driver needs to issue one iteration (ctypes launches + NCCL calls).  When the
host time exceeds the device time the rank is host-bound.

    python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1 \
        tools/strip_rank_probe.py 8 200
"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1409_7474_b200 import _native as N, scenes, default_params, ModelKind, SeedSpec  # noqa: E402
from paper_1409_7474_b200.strips import DeviceStrip, DistComm, StripDriver, plan_strips  # noqa: E402

gpus, iters = int(sys.argv[1]), int(sys.argv[2])
size = 32768
rows = size // gpus
dist.init_process_group("nccl")
torch.cuda.set_device(0)
n_rects = max(1, int(round(20000 * (rows * size) / (32768.0 * 32768.0))))
sc = scenes.config5(size, 20000, iters, rows=(0, rows))
win = plan_strips(rows, size, 1)[0]
prm = default_params(ModelKind.REGION, **sc.params)
strip = DeviceStrip(sc.image, win, SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign), prm)
N.check(N.lib.lse_run_set_option(strip.h, b"skip_uniform", 0))
drv = StripDriver([strip], DistComm(strip))
drv.setup()
drv.advance(20)
strip.synchronize()
N.check(N.lib.lse_run_begin_timing(strip.h))
t0 = time.perf_counter()
for _ in range(iters):
    drv.step()
t_issue = time.perf_counter() - t0
drv.flush()
ms = C.c_double()
N.check(N.lib.lse_run_end_timing(strip.h, C.byref(ms)))
strip.synchronize()
t_wall = time.perf_counter() - t0
print(f"rank share of {gpus} GPUs: {rows}x{size} px, fused={drv.fused}: device "
      f"{1e3 * ms.value / iters:.1f} us/iteration, host issue {1e6 * t_issue / iters:.1f} "
      f"us/iteration, wall {1e6 * t_wall / iters:.1f} us/iteration")
dist.destroy_process_group()
