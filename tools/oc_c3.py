import sys, time, ctypes as C
sys.path.insert(0, "/root/repo")
import numpy as np
import torch  # noqa: F401  (as bench.py)
from paper_1409_7474_b200 import _native as N, scenes, default_params, ModelKind
from paper_1409_7474_b200.bands import BandEvolutionRun
for rep in range(3):
    sc3 = scenes.config3(4096, 1000)
    prm3 = default_params(ModelKind.REGION, **sc3.params)
    run3 = BandEvolutionRun(sc3.image, sc3.extra["signs"], prm3)
    run3.set_native_option("skip_uniform", 0)
    signs3 = np.ascontiguousarray(sc3.extra["signs"], dtype=np.int8)
    init3 = N.LsePhi0()
    init3.kind = N.LSE_PHI0_SIGNS
    init3.signs = signs3.ctypes.data_as(C.POINTER(C.c_byte))
    init3.scale = 1.0
    st3 = N.LseStatus()
    h3 = run3._dev.h
    def job3():
        N.check(N.lib.lse_run_set_state(h3, C.byref(init3)))
        N.check(N.lib.lse_run_advance(h3, sc3.iters, C.byref(st3)))
    for j in range(5):
        ms = C.c_double()
        N.check(N.lib.lse_run_begin_timing(h3))
        job3()
        N.check(N.lib.lse_run_end_timing(h3, C.byref(ms)))
        print(rep, j, round(ms.value, 1), st3.fast_iterations, st3.generic_iterations, flush=True)
    del run3
