import ctypes as C, time, sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_1409_7474_b200 import _native as N, scenes, default_params, ModelKind
from paper_1409_7474_b200.engine import _native_params
size = int(sys.argv[1]); iters = int(sys.argv[2])
sc = scenes.config5_crop(size, iters)
prm = default_params(ModelKind.REGION, **sc.params)
p, keep = _native_params(prm)
polys = np.ascontiguousarray(np.concatenate(sc.polygons)); counts = np.array([len(q) for q in sc.polygons], dtype=np.int64)
init = N.LsePhi0(); init.kind = N.LSE_PHI0_POLYGONS; init.poly_xy = N.dptr(polys)
init.poly_counts = counts.ctypes.data_as(N._llp); init.n_polys = len(counts); init.inside_sign = sc.inside_sign
h = C.c_void_p(); img = np.ascontiguousarray(sc.image)
N.check(N.lib.lse_run_create(C.byref(h), C.byref(p), size, size, img.ctypes.data_as(C.c_void_p), 1, C.byref(init)))
N.check(N.lib.lse_run_set_option(h, b"skip_uniform", 0))
st = N.LseStatus()
prof = len(sys.argv) > 3
if prof:
    N.check(N.lib.lse_run_set_profiling(h, 1))
for rep in range(3):
    N.check(N.lib.lse_run_set_state(h, C.byref(init)))
    t0 = time.perf_counter(); N.check(N.lib.lse_run_begin_timing(h))
    N.check(N.lib.lse_run_advance(h, iters, C.byref(st)))
    ms = C.c_double(); N.check(N.lib.lse_run_end_timing(h, C.byref(ms)))
    print(size, "wall ms/it", (time.perf_counter()-t0)*1e3/iters, "gpu ms/it", ms.value/iters, flush=True)
if prof:
    u, p_, nu, np_ = C.c_double(), C.c_double(), C.c_longlong(), C.c_longlong()
    N.check(N.lib.lse_run_kernel_times(h, C.byref(u), C.byref(nu), C.byref(p_), C.byref(np_)))
    print(size, "update ms", u.value / max(1, nu.value), "partition+finalize ms", p_.value / max(1, np_.value))
