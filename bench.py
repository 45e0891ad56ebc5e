#!/usr/bin/env python
"""Benchmark of the fused LSE iteration on B200 (BASELINE.json metric).

Headline workload (default, `--config C5`; BASELINE.json configs[4], SURVEY.md
section 8d "C5"): one 32768 x 32768 float32 panchromatic scene (1.07 Gpx)
with 20000 seeded rectangles, region-based LSE (R_Td), Gaussian sigma 1.5
(9x9, radius 4), dt = 15, 500 fixed iterations (conv_check_every = 501),
seed box [2048, 30720]^2.  Synthetic data (seeded numpy PCG64) stands in for
the paper's images; inputs (4.3 GB) are larger than L2.

One *step* = one complete extraction job: seed rasterization + partition
init + 500 iterations, inputs resident in HBM (`value`).  `e2e` repeats the
job through the C ABI with host buffers (pinned H2D of the image each step,
D2H of the packed object mask); `e2e_dropin` through the drop-in
`run(image, seeds, params)` with a pageable numpy image, returning the
reference's bool ExtractionResult.mask.

`--config C4 --gpus N`: BASELINE configs[3], 512 seeded 1024^2 8-bit RGB
tiles, region / edge alternating, 300 iterations; tiles k = rank, rank + N,
... per GPU (independent units, no collective), one batch per GPU.

Metric: Gpixel-iterations/s (whole job, all ranks).  Roofline: canonical
algorithmic bytes (read I 4 B + read phi 4 B + write phi 4 B =
12 B/px-it) over the measured device time of one iteration's kernels, against
the measured HBM copy bandwidth in MEASURED_PEAKS.json.  The bit-state design
actually moves ~4.6 B/px-it; both fractions are reported.

`--impl reference` times the CPU restatement of the reference loop
(oracle/lse_oracle.c, bit-exact to lsekit, all host threads) on a bounded
sample of the same workload, with the same `config` as this arm.  It imports
neither the package nor its library.
"""

from __future__ import annotations

import argparse
import ctypes as C
import importlib.util
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))

HBM_FALLBACK_GBS = 6650.0
METRIC = "Gpixel-iterations/s of the LSE update"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=["C5", "C4", "C3", "C2", "C1"], default="C5")
    ap.add_argument("--size", type=int, default=32768, help="C5 scene side (32768)")
    ap.add_argument("--iters", type=int, default=500, help="C5 iterations per job")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--mode", choices=["strips", "replicas"], default="strips",
                    help="C5, N > 1: row strips of one scene (strong scaling) or N replicas")
    ap.add_argument("--strips-n1", action="store_true",
                    help="run the row-strip path (NCCL communicator) even at N = 1 "
                         "(launch under torch.distributed.run)")
    ap.add_argument("--c4-tiles", type=int, default=512,
                    help="C4 tiles (0: skip the other configs of the C5 line)")
    ap.add_argument("--skip-steps", type=int, default=None,
                    help="steps of the uniform-window-skip measurement (default: --steps)")
    ap.add_argument("--dropin-steps", type=int, default=2,
                    help="C5 steps of the drop-in run() end-to-end leg")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


def load_scenes():
    """paper_1409_7474_b200/scenes.py as a stand-alone module (numpy only):
    the reference arm must not import the package or load its library."""
    name = "lse_bench_scenes"
    if name in sys.modules:
        return sys.modules[name]
    spec = importlib.util.spec_from_file_location(
        name, os.path.join(REPO, "paper_1409_7474_b200", "scenes.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


def oracle_modules():
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import lse_oracle as O
    import lse_oracle_c as OC
    return O, OC


# ----------------------------------------------------------- config strings
def c5_config(args, ws, strips):
    return {"workload": f"C5: {args.size}x{args.size} region LSE, 20000-rect density, sigma 1.5 "
                        f"(9x9), dt 15, {args.iters} fixed iterations per step",
            "parallelism": (f"row strips x{ws} (NCCL halo + partial allgather)"
                            if strips else f"replicas x{ws}" if ws > 1 else "single GPU"),
            "l2": "inputs (4.3 GB image) larger than L2"}


def c4_config(args, ws):
    return {"workload": f"C4: {args.c4_tiles} seeded 1024^2 8-bit RGB tiles (luma on device), "
                        "even tiles region / odd tiles edge, sigma 1.0, dt 15, 300 fixed "
                        "iterations per step",
            "parallelism": f"tiles k::{ws} per GPU, one batch per GPU, no collective",
            "l2": "inputs (512 x 4 MB luma planes) larger than L2"}


def small_config(name, ws):
    d = {"C1": "C1: 256^2 region, dt 100, sigma 1 (5x5), 200 fixed iterations per step",
         "C2": "C2: 1024^2 edge (sigma1 1.5, gain 255), sigma 1 (9x9), dt 15, 500 fixed "
               "iterations per step",
         "C3": "C3: 4096^2 x 4 bands (fp32), vector region term, +-1 checkerboard of 64^2 "
               "cells, sigma 1 (9x9), dt 15, 1000 fixed iterations per step"}[name]
    return {"workload": d, "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
            "l2": "C1/C2 L2-resident (one resident kernel per job: barrier / dependency-latency bound); C3 inputs 268 MB > L2"
            if name != "C3" else "inputs (268 MB of bands) larger than L2"}


# ----------------------------------------------------------------- CPU side
class CpuSample:
    """A bounded sample of one BASELINE workload on the C restatement of the
    reference loop (oracle/lse_oracle.c, bit-exact to lsekit); each step()
    advances `its` iterations and returns the pixel-iterations done."""

    def __init__(self, config, threads=0, its=None):
        O, OC = oracle_modules()
        sc = load_scenes()
        OC.set_threads(threads)
        self.threads = OC.load().oracle_threads()
        self.runs = []

        def prm(s):
            p = s.params
            return O.OracleParams(model=s.model, dt=p["dt"], sigma2=p["sigma2"],
                                  ts_reg=p["ts_reg"], max_iters=10 ** 7,
                                  conv_check_every=10 ** 7 + 1,
                                  sigma1=p.get("sigma1", 1.0), ts_pre=p.get("ts_pre", 9),
                                  edge_gain=p.get("edge_gain", 255.0))

        if config == "C5":
            size = 2048
            s = sc.config5_crop(size, 10 ** 6)
            phi0 = O.rasterize_seeds(list(s.polygons), s.inside_sign, size, size)
            self.runs = [OC.COracleRun(s.image.astype(np.float64), phi0, prm(s),
                                       O.gaussian_weights)]
            self.its = its or 20
            self.desc = f"C5-density crop {size}x{size} (1/256 of the scene)"
        elif config == "C4":
            for k in range(16):
                s = sc.config4_tile(k, 1024, 300)
                phi0 = O.rasterize_seeds(list(s.polygons), s.inside_sign, 1024, 1024)
                self.runs.append(OC.COracleRun(sc.luma(s.image), phi0, prm(s),
                                               O.gaussian_weights))
            self.its = its or 2
            self.desc = "C4 tiles 0..15 (of 512), one after another"
        elif config == "C3":
            s = sc.config3(4096, 10 ** 6)
            self.runs = [OC.COracleRun(s.image.astype(np.float64),
                                       s.extra["signs"].astype(np.float64), prm(s),
                                       O.gaussian_weights)]
            self.its = its or 2
            self.desc = "C3 4096^2 x 4 bands (multi-band restatement of the reference step)"
        else:
            s = sc.config1() if config == "C1" else sc.config2()
            h, w = s.image.shape
            phi0 = O.rasterize_seeds(list(s.polygons), s.inside_sign, w, h)
            self.runs = [OC.COracleRun(s.image.astype(np.float64), phi0, prm(s),
                                       O.gaussian_weights)]
            self.its = its or (200 if config == "C1" else 50)
            self.desc = f"{config} full image"
        self.npx = sum(r.image.shape[-2] * r.image.shape[-1] for r in self.runs)

    def step(self):
        for r in self.runs:
            r.advance(self.its)
        return self.npx * self.its


def cpu_rate(config, seconds, threads=0):
    """Gpix-it/s of the CPU restatement on a bounded sample of `config`."""
    s = CpuSample(config, threads)
    s.step()                                   # warm-up (page faults, allocations)
    t0 = time.perf_counter()
    n = 0
    while True:
        n += s.step()
        dt = time.perf_counter() - t0
        if dt >= seconds:
            break
    core = "1 core (the reference is single-threaded)" if threads == 1 else \
        f"{s.threads} threads"
    return {"value": n / dt / 1e9, "unit": "Gpix-it/s", "cores": s.threads, "kind": "port",
            "sample": f"{s.desc}: {n // s.npx} iterations in {dt:.1f} s, {core} "
                      "(oracle/lse_oracle.c, bit-exact C restatement of lsekit)"}


def run_reference(args, ws, rank):
    """--impl reference: the CPU restatement of the reference path, bounded
    sample of the arm's workload, all host threads; rank 0 only."""
    if rank != 0:
        return
    cfg = args.config
    s = CpuSample(cfg, 0)
    for _ in range(args.warmup):
        s.step()
    t0 = time.perf_counter()
    n = 0
    for _ in range(args.steps):
        n += s.step()
    dt = time.perf_counter() - t0
    val = n / dt / 1e9
    if cfg == "C5":
        config = c5_config(args, ws, ws > 1 and args.mode == "strips")
    elif cfg == "C4":
        config = c4_config(args, ws)
    else:
        config = small_config(cfg, ws)
    sample = f"{s.desc} x {s.its} its per step x {args.steps} steps"
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "Gpix-it/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong" if cfg == "C5" and ws > 1 and args.mode == "strips" else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE statistics)", "config": config,
        "cpu_baseline": {"value": val, "unit": "Gpix-it/s", "cores": s.threads, "kind": "port",
                         "sample": sample + " (oracle/lse_oracle.c; the reference package "
                                            "cannot travel to the GPU box)"},
        "e2e": {"value": val, "unit": "Gpix-it/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.proc = None
        self.f = None

    def start(self):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.n0 = 0
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        # the sampler is live (first sample written) before the timed region starts;
        # samples taken before it are not counted
        t0 = time.time()
        while time.time() - t0 < 5.0 and self.proc.poll() is None:
            self.n0 = len(self._lines())
            if self.n0:
                break
            time.sleep(0.02)

    def _lines(self):
        with open(self.f.name) as fh:
            return [ln for ln in fh.read().splitlines() if ln.count(",") == 5]

    def stop(self):
        if self.proc is None:
            return None
        window = "timed region"
        if len(self._lines()) <= self.n0:
            # a timed region shorter than the sampling period: take the first
            # sample after it (the clocks have not dropped yet)
            window = "first sample after a short timed region"
            t0 = time.time()
            while time.time() - t0 < 1.0 and len(self._lines()) <= self.n0:
                time.sleep(0.01)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in self._lines()[self.n0:]:
            parts = [x.strip() for x in line.split(",")]
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2:]))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for _, _, r in rows for k, v in enumerate(r)
                          if v.lower().startswith("active")})
        loaded = [s for s, _, _ in rows if s > 200] or [s for s, _, _ in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(m for _, m, _ in rows),
                "reasons": reasons, "samples": len(rows), "window": window}


class Dist:
    """Barrier / max-over-ranks helpers (one process per GPU)."""

    def __init__(self, dist):
        self.dist = dist

    def barrier(self):
        import torch
        if self.dist is not None:
            self.dist.barrier()
        torch.cuda.synchronize()

    def max(self, x):
        import torch
        if self.dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


# ------------------------------------------------- the other BASELINE configs
def small_job(name, steps):
    """C1 / C2 (single small images: L2-resident, one resident kernel per job) and C3
    (4096^2 x 4 bands): device time of the fixed-iteration evolution through
    the C ABI, inputs resident, dense pass.  Returns (Gpix-it/s, ms/job,
    px-its per job, launches per job)."""
    from paper_1409_7474_b200 import _native as N, scenes
    from paper_1409_7474_b200 import default_params, ModelKind, SeedSpec
    from paper_1409_7474_b200.engine import _native_params, _phi0_polygons
    import warnings
    if name == "C3":
        from paper_1409_7474_b200.bands import BandEvolutionRun
        sc = scenes.config3(4096, 1000)
        prm = default_params(ModelKind.REGION, **sc.params)
        run = BandEvolutionRun(sc.image, sc.extra["signs"], prm)
        run.set_native_option("skip_uniform", 0)
        signs = np.ascontiguousarray(sc.extra["signs"], dtype=np.int8)
        init = N.LsePhi0()
        init.kind = N.LSE_PHI0_SIGNS
        init.signs = signs.ctypes.data_as(C.POINTER(C.c_byte))
        init.scale = 1.0
        h = run._dev.h
        keep = (run, signs)
        npx, iters = 4096 * 4096, sc.iters
    else:
        sc = scenes.config1() if name == "C1" else scenes.config2()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            prm = default_params(ModelKind.from_name(sc.model), **sc.params)
        p, pkeep = _native_params(prm)
        init, ikeep = _phi0_polygons(SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign))
        img = np.ascontiguousarray(sc.image)
        h = C.c_void_p()
        N.check(N.lib.lse_run_create(C.byref(h), C.byref(p), img.shape[0], img.shape[1],
                                     img.ctypes.data_as(C.c_void_p), 1, C.byref(init)))
        N.check(N.lib.lse_run_set_option(h, b"skip_uniform", 0))
        keep = (pkeep, ikeep, img)
        npx, iters = img.size, sc.iters
    st = N.LseStatus()

    def job():
        N.check(N.lib.lse_run_set_state(h, C.byref(init)))
        N.check(N.lib.lse_run_advance(h, iters, C.byref(st)))

    for _ in range(3):                  # warm-up (module load, clocks back up)
        job()
    ms = C.c_double()
    l0 = N.lib.lse_launch_count()
    N.check(N.lib.lse_run_begin_timing(h))
    for _ in range(steps):
        job()
    N.check(N.lib.lse_run_end_timing(h, C.byref(ms)))
    launches = (N.lib.lse_launch_count() - l0) / steps
    assert st.iteration == iters, st.iteration
    if name != "C3":
        N.lib.lse_run_destroy(h)
    del keep
    return npx * iters * steps / (ms.value / 1e3) / 1e9, ms.value / steps, npx * iters, launches


class C4Job:
    """This rank's share of the C4 tiles as one device batch."""

    def __init__(self, n_tiles, rank, ws):
        from concurrent.futures import ProcessPoolExecutor
        from paper_1409_7474_b200 import _native as N
        from paper_1409_7474_b200 import default_params, ModelKind, SeedSpec
        from paper_1409_7474_b200.batch import TileBatch, _tile_run, shard
        from paper_1409_7474_b200.engine import _phi0_polygons
        sc = load_scenes()
        self.N = N
        self.mine = shard(n_tiles, rank, ws)
        t0 = time.perf_counter()
        with ProcessPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
            self.scenes = list(ex.map(sc.config4_tile, self.mine, chunksize=4))
        self.t_gen = time.perf_counter() - t0
        self.seeds = [SeedSpec(polygons=s.polygons, inside_sign=s.inside_sign)
                      for s in self.scenes]
        self.params = [default_params(ModelKind.from_name(s.model), **s.params)
                       for s in self.scenes]
        t0 = time.perf_counter()
        self.runs = [_tile_run(s.image, sd, p)
                     for s, sd, p in zip(self.scenes, self.seeds, self.params)]
        self.t_create = time.perf_counter() - t0
        self.inits = [_phi0_polygons(sd) for sd in self.seeds]
        for r in self.runs:
            r.set_native_option("skip_uniform", 0)
        self.tb = TileBatch(self.runs)
        self.npx = len(self.mine) * 1024 * 1024

    def reset(self):
        for r, (init, _) in zip(self.runs, self.inits):
            self.N.check(self.N.lib.lse_run_set_state(r._dev.h, C.byref(init)))

    def job(self):
        self.tb.advance(300)

    def close(self):
        self.tb.close()
        self.runs = None


def other_configs(steps, c4_tiles, cpu_seconds, with_cpu):
    """C1 / C2 / C3 / C4 measured alongside the C5 headline (1 GPU), each with
    its CPU baseline (C1 / C2 on 1 core as the reference runs, C3 / C4 on all
    host threads)."""
    import torch
    out = {}
    peak, _ = measured_peaks()
    v3, ms3, _, l3 = small_job("C3", steps)
    out["C3"] = {"value": v3, "unit": "Gpix-it/s", "ms_per_job": ms3, "launches_per_job": l3,
                 "workload": small_config("C3", 1)["workload"],
                 "roofline": {"bound": "hbm", "algorithmic_bytes_per_px_it": 24.0,
                              "achieved": v3 * 24.0, "peak": peak, "unit": "GB/s",
                              "frac": v3 * 24.0 / peak}}
    if c4_tiles > 0:
        j = C4Job(c4_tiles, 0, 1)
        j.reset()
        j.job()                                             # warm-up
        N = j.N
        N.check(N.lib.lse_batch_set_timing(j.tb.h, 1))
        for _ in range(steps):
            j.reset()
            torch.cuda.synchronize()
            j.job()
        ms, calls = C.c_double(), C.c_longlong()
        N.check(N.lib.lse_batch_elapsed(j.tb.h, C.byref(ms), C.byref(calls)))
        v4 = j.npx * 300 * calls.value / (ms.value / 1e3) / 1e9
        out["C4"] = {"value": v4, "unit": "Gpix-it/s", "ms_per_job": ms.value / calls.value,
                     "tiles": c4_tiles,
                     "roofline": {"bound": "hbm", "algorithmic_bytes_per_px_it": 12.0,
                                  "achieved": v4 * 12.0, "peak": peak, "unit": "GB/s",
                                  "frac": v4 * 12.0 / peak},
                     "workload": c4_config(argparse.Namespace(c4_tiles=c4_tiles), 1)["workload"],
                     "tile_gen_s": round(j.t_gen, 1), "tile_setup_s": round(j.t_create, 1)}
        j.close()
    for name in ("C1", "C2"):
        v, ms, _, launches = small_job(name, steps)
        out[name] = {"value": v, "unit": "Gpix-it/s", "ms_per_job": ms,
                     "launches_per_job": launches,
                     "workload": small_config(name, 1)["workload"],
                     "bound": "barrier + dependency latency of the resident kernel (k_resident: one launch per job; not HBM)"}
    if with_cpu:
        for name, thr in (("C1", 1), ("C2", 1), ("C3", 0), ("C4", 0)):
            if name in out:
                cb = cpu_rate(name, min(cpu_seconds, 8.0), thr)
                out[name]["cpu_baseline"] = cb
    return out


# ------------------------------------------------------------------ C4 line
def main_c4(args, ws, rank, local, dist):
    import torch
    D = Dist(dist)
    j = C4Job(args.c4_tiles, rank, ws)
    N = j.N
    for _ in range(args.warmup):
        j.reset()
        j.job()
    N.check(N.lib.lse_batch_set_timing(j.tb.h, 1))
    clocks = ClockSampler(local)
    D.barrier()
    clocks.start()
    launches = 0
    for _ in range(args.steps):
        j.reset()                        # seeds re-rasterized outside the timed region
        torch.cuda.synchronize()
        l0 = N.lib.lse_launch_count()
        j.job()
        launches += N.lib.lse_launch_count() - l0
    D.barrier()
    clk = clocks.stop()
    ms, calls = C.c_double(), C.c_longlong()
    N.check(N.lib.lse_batch_elapsed(j.tb.h, C.byref(ms), C.byref(calls)))
    t_ms = D.max(ms.value)
    total_px_its = args.c4_tiles * 1024 * 1024 * 300 * args.steps
    value = total_px_its / (t_ms / 1e3) / 1e9
    its = [r.state.iteration for r in j.runs]
    assert all(i == 300 for i in its), its
    # end to end through the public API: run_tiles on host uint8 tiles -> masks
    e2e = None
    if not args.no_e2e:
        from paper_1409_7474_b200.batch import run_tiles
        imgs = [s.image for s in j.scenes]
        j.close()
        run_tiles(imgs[:2], j.seeds[:2], j.params[:2])       # warm-up
        D.barrier()
        t0 = time.perf_counter()
        for _ in range(max(1, min(args.steps, 2))):
            res = run_tiles(imgs, j.seeds, j.params)
        torch.cuda.synchronize()
        e_s = D.max((time.perf_counter() - t0) / max(1, min(args.steps, 2)))
        assert all(r.iterations == 300 for r in res)
        e2e = {"value": args.c4_tiles * 1024 * 1024 * 300 / e_s / 1e9, "unit": "Gpix-it/s",
               "h2d_bytes_per_step": sum(i.nbytes for i in imgs),
               "d2h_bytes_per_step": sum(r.mask.nbytes for r in res),
               "ms_per_step": e_s * 1e3,
               "path": "batch.run_tiles(uint8 RGB host tiles) -> ExtractionResult.mask (bool), "
                       "wall clock incl. run creation, H2D, decode, 300 its, D2H"}
    else:
        j.close()
    peak, peak_kind = measured_peaks()
    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            cpu = cpu_rate("C4", args.cpu_seconds)
        line = {
            "metric": METRIC, "value": value, "unit": "Gpix-it/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "higher_is_better": True, "mode": "dense (skip_uniform=0)", "scaling": "weak",
            "vs_baseline": None, "dtype": "f32+f64-guard (bit state)",
            "data": "synthetic (seeded, BASELINE C4 statistics; 512 distinct tiles)",
            "config": c4_config(args, ws),
            "roofline": {"bound": "hbm", "kernel": "one batched iteration (update + partition "
                                                  "+ finalize) incl. gather/scatter",
                         "achieved": 12.0 * value, "peak": peak, "unit": "GB/s",
                         "frac": 12.0 * value / peak, "traffic": None,
                         "peak_source": peak_kind, "algorithmic_bytes_per_px_it": 12.0},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk, "tiles_per_gpu": len(j.mine),
        }
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ C5 line
def build_c5(args, ws, rank, strips):
    """The measured job: one strip of the scene per rank (strips) or the whole
    scene per rank (replicas / N = 1)."""
    import torch
    from types import SimpleNamespace
    from paper_1409_7474_b200 import _native as N, scenes
    from paper_1409_7474_b200.engine import _native_params
    from paper_1409_7474_b200 import default_params, ModelKind, SeedSpec
    from paper_1409_7474_b200.strips import DeviceStrip, DistComm, StripDriver, plan_strips
    n_rects = max(1, int(round(20000 * (args.size / 32768.0) ** 2)))
    jb = SimpleNamespace(strips=strips)
    win = plan_strips(args.size, args.size, ws)[rank] if strips else None
    t0 = time.perf_counter()
    sc = scenes.config5(size=args.size, n_rects=n_rects, iters=args.iters,
                        seed_offset=0 if strips else rank,
                        rows=(win.y_lo, win.y_hi) if strips else None)
    jb.t_gen = time.perf_counter() - t0
    jb.Hl, jb.W = sc.image.shape           # local rows (a strip: owned + halo rows)
    jb.npx_local = jb.Hl * jb.W
    prm = default_params(ModelKind.REGION, **sc.params)
    jb.prm, jb.polygons, jb.inside = prm, sc.polygons, sc.inside_sign
    p, jb.keep_w = _native_params(prm)
    # pinned host copies for the end-to-end leg
    img_pin = torch.empty((jb.Hl, jb.W), dtype=torch.float32, pin_memory=True)
    img_pin.numpy()[...] = sc.image
    jb.nbytes_mask = (jb.npx_local + 7) // 8
    mask_pin = torch.empty(jb.nbytes_mask, dtype=torch.uint8, pin_memory=True)
    jb.img_pin, jb.mask_pin = img_pin, mask_pin
    polys = np.ascontiguousarray(np.concatenate(sc.polygons), dtype=np.float64)
    counts = np.ascontiguousarray([len(q) for q in sc.polygons], dtype=np.int64)
    jb.poly_bytes = polys.nbytes + counts.nbytes
    jb.st = st = N.LseStatus()
    inside = sc.inside_sign
    del sc.image
    if strips:
        # one row strip of the scene per rank; halo rows + partials over NCCL
        strip = DeviceStrip(img_pin.numpy(), win, SeedSpec(polygons=jb.polygons,
                                                           inside_sign=inside), prm)
        drv = StripDriver([strip], DistComm(strip))
        drv.share_image_range()
        jb.strip, jb.drv, jb.h = strip, drv, strip.h

        def job():
            strip.reset()
            drv.initialize()
            s0 = drv.advance(args.iters)[0]
            assert s0.iteration == args.iters, s0.iteration
            st.exact_fallbacks = s0.exact_fallbacks

        def job_e2e():
            strip.load_image(img_pin.data_ptr(), True)
            drv.share_image_range()
            job()
            N.check(N.lib.lse_run_read_mask(jb.h, C.cast(C.c_void_p(mask_pin.data_ptr()),
                                                         C.POINTER(C.c_ubyte)), inside, 1))

        def close():
            jb.drv = jb.strip = None
    else:
        init = N.LsePhi0()
        init.kind = N.LSE_PHI0_POLYGONS
        init.poly_xy = N.dptr(polys)
        init.poly_counts = counts.ctypes.data_as(N._llp)
        init.n_polys = len(counts)
        init.inside_sign = inside
        jb.keep_init = (init, polys, counts)
        h = C.c_void_p()
        N.check(N.lib.lse_run_create(C.byref(h), C.byref(p), jb.Hl, jb.W,
                                     C.c_void_p(img_pin.data_ptr()), 1, C.byref(init)))
        jb.h = h

        def job():
            N.check(N.lib.lse_run_set_state(h, C.byref(init)))
            N.check(N.lib.lse_run_advance(h, args.iters, C.byref(st)))
            assert st.iteration == args.iters, st.iteration

        def job_e2e():
            N.check(N.lib.lse_run_load_image(h, C.c_void_p(img_pin.data_ptr()), 1))
            job()
            N.check(N.lib.lse_run_read_mask(h, C.cast(C.c_void_p(mask_pin.data_ptr()),
                                                      C.POINTER(C.c_ubyte)), inside, 1))

        def close():
            N.lib.lse_run_destroy(h)
    jb.job, jb.job_e2e, jb.close = job, job_e2e, close
    return jb


def main_c5(args, ws, rank, local, dist):
    import torch
    from paper_1409_7474_b200 import _native as N
    D = Dist(dist)
    strips = (ws > 1 and args.mode == "strips") or args.strips_n1
    jb = build_c5(args, ws, rank, strips)      # a failure here is fatal on every rank
    h, job, job_e2e, st = jb.h, jb.job, jb.job_e2e, jb.st
    npx = args.size * args.size
    # whole-job pixel-iterations per step (all ranks): strips share one scene,
    # replicas each run their own
    job_px_its = npx * args.iters * (1 if strips else ws)

    # ---- dense pass (every pixel recomputed every iteration): the headline
    N.check(N.lib.lse_run_set_option(h, b"skip_uniform", 0))
    for _ in range(args.warmup):
        job()
    clocks = ClockSampler(local)
    D.barrier()
    clocks.start()
    N.check(N.lib.lse_run_set_profiling(h, 1))
    launches0 = N.lib.lse_launch_count()
    N.check(N.lib.lse_run_begin_timing(h))
    for _ in range(args.steps):
        job()
    ms = C.c_double()
    N.check(N.lib.lse_run_end_timing(h, C.byref(ms)))
    launches = N.lib.lse_launch_count() - launches0
    D.barrier()
    clk = clocks.stop()
    t_ms = D.max(ms.value)
    upd_ms, part_ms = C.c_double(), C.c_double()
    n_upd, n_part = C.c_longlong(), C.c_longlong()
    N.check(N.lib.lse_run_kernel_times(h, C.byref(upd_ms), C.byref(n_upd), C.byref(part_ms),
                                       C.byref(n_part)))
    N.check(N.lib.lse_run_set_profiling(h, 0))
    fallbacks = st.exact_fallbacks
    spec = (C.c_longlong * 4)()
    N.check(N.lib.lse_run_spec_stats(h, spec))
    spec_stats = {"fused_iterations": int(spec[0]), "redone": int(spec[1]),
                  "fix_list_pixels": int(spec[2]), "enabled": bool(spec[3]),
                  "note": "cumulative over the run's jobs (warm-up included): one-pass "
                          "speculative iterations, of which redone whole (prediction outside "
                          "its band), pixels decided from the fix list"}
    px_its = job_px_its * args.steps
    value = px_its / (t_ms / 1e3) / 1e9

    # ---- same jobs with the exact uniform-window skip (product default)
    skip_steps = args.steps if args.skip_steps is None else args.skip_steps
    skip = None
    if skip_steps > 0:
        N.check(N.lib.lse_run_set_option(h, b"skip_uniform", 1))
        job()
        D.barrier()
        N.check(N.lib.lse_run_set_profiling(h, 1))
        N.check(N.lib.lse_run_begin_timing(h))
        for _ in range(skip_steps):
            job()
        N.check(N.lib.lse_run_end_timing(h, C.byref(ms)))
        D.barrier()
        s_ms = D.max(ms.value)
        su, sp, nsu, nsp = C.c_double(), C.c_double(), C.c_longlong(), C.c_longlong()
        N.check(N.lib.lse_run_kernel_times(h, C.byref(su), C.byref(nsu), C.byref(sp),
                                           C.byref(nsp)))
        N.check(N.lib.lse_run_set_profiling(h, 0))
        skip = {"value": job_px_its * skip_steps / (s_ms / 1e3) / 1e9,
                "unit": "Gpix-it/s", "ms_per_step": s_ms / skip_steps,
                "update_ms": su.value / max(1, nsu.value),
                "partition_ms": sp.value / max(1, nsp.value),
                "note": "skip_uniform=1: warp blocks whose whole stencil window is uniform "
                        "are copied (|grad phi| == 0 there, so u == phi exactly); results "
                        "bit-identical to the dense pass"}
        N.check(N.lib.lse_run_set_option(h, b"skip_uniform", 0))

    # ---- end to end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        job_e2e()
        D.barrier()
        N.check(N.lib.lse_run_begin_timing(h))
        for _ in range(args.steps):
            job_e2e()
        N.check(N.lib.lse_run_end_timing(h, C.byref(ms)))
        D.barrier()
        e_ms = D.max(ms.value)
        e2e = {"value": px_its / (e_ms / 1e3) / 1e9, "unit": "Gpix-it/s",
               "h2d_bytes_per_step": jb.npx_local * 4 + jb.poly_bytes,
               "d2h_bytes_per_step": jb.nbytes_mask, "ms_per_step": e_ms / args.steps,
               "path": "C ABI: pinned float32 image H2D, 500 its, packed mask D2H "
                       "(device events on the run's stream)"}
    jb.close()

    # ---- end to end through the drop-in run() (1 GPU): pageable numpy image
    # in, the reference's bool ExtractionResult.mask out, dense pass
    dropin = None
    if not args.no_e2e and not strips and args.dropin_steps > 0:
        import paper_1409_7474_b200 as L
        os.environ["LSE_SKIP_UNIFORM"] = "0"
        img = np.array(jb.img_pin.numpy())                  # pageable copy
        seeds = L.SeedSpec(polygons=jb.polygons, inside_sign=jb.inside)
        res = L.run(img, seeds, jb.prm)                     # warm-up (one-time staging buffers)
        D.barrier()
        t0 = time.perf_counter()
        for _ in range(args.dropin_steps):
            res = L.run(img, seeds, jb.prm)
        torch.cuda.synchronize()
        d_s = D.max((time.perf_counter() - t0) / args.dropin_steps)
        del os.environ["LSE_SKIP_UNIFORM"]
        assert res.iterations == args.iters and res.mask.dtype == np.bool_
        dropin = {"value": job_px_its / d_s / 1e9, "unit": "Gpix-it/s",
                  "h2d_bytes_per_step": img.nbytes, "d2h_bytes_per_step": res.mask.nbytes,
                  "ms_per_step": d_s * 1e3,
                  "path": "paper_1409_7474_b200.run(numpy float32 pageable image, SeedSpec, "
                          "EvolutionParams) -> ExtractionResult.mask (bool, 1 B/px); wall "
                          "clock incl. run creation and teardown, dense pass; one untimed warm-up call"}

    # ---- roofline of one iteration.  Fused runs: k_update_fused (the partition
    # of b^n and the update b^n -> b^{n+1} in one pass) is the dominant kernel,
    # the finalize / fix / redo launches are 'partition_ms'; two-pass runs
    # (strips): k_update + k_partition (+ finalize)
    peak, peak_kind = measured_peaks()
    t_upd = upd_ms.value / max(1, n_upd.value)
    t_part = part_ms.value / max(1, n_part.value)
    t_iter = t_upd + t_part
    fused = bool(spec[3])
    canon = 12.0 * jb.npx_local       # this rank's pixels per iteration
    # bytes actually moved per pixel-iteration: the fp32 data plane, b in and
    # out, P read (fused: one pass); two-pass: + b and P again in the partition
    actual = ((4.0 + 3.0 / 8.0) if fused else (4.0 + 2.0 / 8.0 + 3.0 / 8.0)) * jb.npx_local
    traffic = None
    tp = os.path.join(REPO, "profiles", "traffic_latest.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                td = json.load(f)
            if int(td.get("size", 0)) == args.size and ws == 1:
                traffic = float(td["bytes_per_iteration"])
        except Exception:
            traffic = None
    roof = {"bound": "hbm",
            "kernel": ("k_update_fused + finalize + fix (one-pass speculative LSE iteration)"
                       if fused else "k_update + k_partition (+ finalize): one LSE iteration"),
            "achieved": canon / (t_iter / 1e3) / 1e9 if t_iter > 0 else None,
            "peak": peak, "unit": "GB/s",
            "frac": (canon / (t_iter / 1e3) / 1e9) / peak if t_iter > 0 else None,
            "traffic": traffic, "peak_source": peak_kind,
            "algorithmic_bytes_per_px_it": 12.0, "actual_bytes_per_px_it": actual / jb.npx_local,
            "achieved_actual_gbs": actual / (t_iter / 1e3) / 1e9 if t_iter > 0 else None,
            "frac_actual": (actual / (t_iter / 1e3) / 1e9) / peak if t_iter > 0 else None,
            "update_ms": t_upd, "partition_ms": t_part,
            "update_share_of_iteration": t_upd / t_iter if t_iter > 0 else None}

    others = None
    if rank == 0 and ws == 1 and args.c4_tiles > 0:
        others = other_configs(max(1, min(args.steps, 3)), args.c4_tiles, args.cpu_seconds,
                               not args.no_cpu_baseline)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_rate("C5", args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value,
            "unit": "Gpix-it/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "mode": "dense (skip_uniform=0: every pixel recomputed every iteration)",
            "scaling": "strong" if strips else "weak", "vs_baseline": None,
            "dtype": "f32+f64-guard (bit state)",
            "data": "synthetic (seeded, BASELINE C5 statistics)",
            "config": c5_config(args, ws, strips),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "e2e_dropin": dropin,
            "gpu_launches": int(launches),
            "uniform_skip": skip, "other_configs": others,
            "clocks": clk, "exact_fallbacks": int(fallbacks), "speculation": spec_stats,
            "scene_gen_s": round(jb.t_gen, 2),
        }
        print(json.dumps(line), flush=True)


def main_small(args, ws, rank, local, dist):
    """--config C1 / C2 / C3: one image per GPU (replicas at N > 1)."""
    D = Dist(dist)
    clocks = ClockSampler(local)
    D.barrier()
    clocks.start()
    v, ms, pxits, launches = small_job(args.config, args.steps)
    D.barrier()
    clk = clocks.stop()
    t_ms = D.max(ms * args.steps)
    value = pxits * ws * args.steps / (t_ms / 1e3) / 1e9
    peak, peak_kind = measured_peaks()
    bpp = 24.0 if args.config == "C3" else 12.0
    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            cpu = cpu_rate(args.config, args.cpu_seconds, 0 if args.config == "C3" else 1)
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "Gpix-it/s", "n_gpus": ws,
            "steps": args.steps, "warmup": 3, "ms_per_step": t_ms / args.steps,
            "higher_is_better": True, "mode": "dense (skip_uniform=0)", "scaling": "weak",
            "vs_baseline": None, "dtype": "f32+f64-guard (bit state)",
            "data": "synthetic (seeded, BASELINE statistics)",
            "config": small_config(args.config, ws),
            "roofline": {"bound": "hbm" if args.config == "C3" else "latency",
                         "kernel": "one LSE iteration", "achieved": bpp * value, "peak": peak,
                         "unit": "GB/s", "frac": bpp * value / peak, "traffic": None,
                         "peak_source": peak_kind, "algorithmic_bytes_per_px_it": bpp},
            "cpu_baseline": cpu, "e2e": None, "gpu_launches": int(launches * args.steps),
            "clocks": clk}), flush=True)


# ----------------------------------------------------------------- GPU side
def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, ws, rank)
    sys.path.insert(0, REPO)
    import torch
    torch.cuda.set_device(local)
    dist = None
    if ws > 1 or args.strips_n1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        if args.config == "C5":
            main_c5(args, ws, rank, local, dist)
        elif args.config == "C4":
            main_c4(args, ws, rank, local, dist)
        else:
            main_small(args, ws, rank, local, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
