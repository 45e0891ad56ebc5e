"""C3 as the bench measures it: set_state(signs) + advance(iters) per job."""
import ctypes as C
import sys
import time
sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import paper_1409_7474_b200 as L  # noqa: E402
from paper_1409_7474_b200 import _native as N, scenes  # noqa: E402
from paper_1409_7474_b200.bands import BandEvolutionRun  # noqa: E402
size, iters = int(sys.argv[1]), int(sys.argv[2])
sc = scenes.config3(size, iters)
run = BandEvolutionRun(sc.image, sc.extra["signs"], L.default_params(L.ModelKind.REGION, **sc.params))
run.set_native_option("skip_uniform", 0)
signs = np.ascontiguousarray(sc.extra["signs"], dtype=np.int8)
init = N.LsePhi0()
init.kind = N.LSE_PHI0_SIGNS
init.signs = signs.ctypes.data_as(C.POINTER(C.c_byte))
init.scale = 1.0
st = N.LseStatus()
import subprocess  # noqa: E402
for j in range(int(sys.argv[3]) if len(sys.argv) > 3 else 4):
    t0 = time.perf_counter()
    ms = C.c_double()
    N.check(N.lib.lse_run_begin_timing(run._dev.h))
    N.check(N.lib.lse_run_set_state(run._dev.h, C.byref(init)))
    N.check(N.lib.lse_run_advance(run._dev.h, iters, C.byref(st)))
    N.check(N.lib.lse_run_end_timing(run._dev.h, C.byref(ms)))
    dt = time.perf_counter() - t0
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks_event_reasons.active",
                          "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    print(f"   events {ms.value:.1f} ms, clock {clk}")
    print(f"job {j}: {dt*1e3:.1f} ms, {dt/iters*1e3:.3f} ms/it, it {st.iteration}, "
          f"fast {st.fast_iterations} generic {st.generic_iterations} fallbacks {st.exact_fallbacks}")
