#!/usr/bin/env python
"""Benchmark: setup + solve of the BASELINE workload on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

A step is one full pass of the hot path: setup_hierarchy (strength, MIS(2), aggregation,
transfer, Galerkin sort/segmented reduce, smoother setup, coarse LU) followed by the
preconditioned Krylov solve to 1e-8, on the configuration BASELINE.json's metric is
quoted on (configs[1]: 3-D 7-point Poisson 256^3, PCG + hybrid K-cycle, fp64).

  value   DOF/s of setup+solve with the matrix already resident in HBM (device generator),
          device time on the library stream, max over ranks.
  e2e     the same metric through the host C-ABI entry point aggmg_setup_and_solve: host
          CSR in, x out, H2D/D2H copies inside the timed region.
  roofline  level-0 damped-Jacobi sweep (the dominant kernel, see profiles/): algorithmic
          bytes per launch / CUDA-event launch time vs MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline  the unmodified reference (oracle/_ref) on all host cores, bounded sample.

Multi-GPU (--gpus N > 1; launched by torchrun, or by bench.py itself when WORLD_SIZE is
unset): the ROW-PARTITIONED solver.  Weak scaling (default) keeps the config's
problem per GPU and doubles the grid along x, then y, then z (256^3 on 1 GPU,
512x256x256 on 2, 512x512x256 on 4, 512^3 on 8); --scaling strong keeps the config's grid
(e.g. --config c5: 512^3 on every N).  Each rank generates and owns one z-slab, setup and solve
exchange halos and scalars over NCCL, coarse levels are agglomerated on rank 0.  --mode
replicas instead runs N independent copies; --emulate-ranks R runs the partitioned path as R
rank threads on one GPU (a transport/overhead diagnostic, not a scaling number).

--impl reference times the reference CPU implementation (oracle/_ref: the unmodified reference
sources compiled by oracle/Makefile) on all host cores, on the SAME configuration: every timed
step is one full setup + solve of the config's grid (the warm-up steps use a 64^3 grid of the
same class, to keep the arm within the driver's budget).  Both arms print the same `config`.
"""
import argparse
import ctypes as C
import datetime
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (label, dims, nx, ny, nz, eps, alpha, method, restart)
    "c1": ("2D 5-point Poisson 512x512, PCG + K-cycle to 1e-8", 2, 512, 512, 1, 1.0, 0.25, "pcg"),
    "c2": ("3D 7-point Poisson 256^3 (16.7M unknowns), PCG + K-cycle AMG to 1e-8, fp64", 3, 256,
           256, 256, 1.0, 0.5, "pcg"),
    "c3": ("3D anisotropic 7-point (eps=1e-3) 384^3, FGMRES(30) + K-cycle to 1e-8", 3, 384, 384,
           384, 1e-3, 0.5, "fgmres"),
    "c4": ("3D variable-coefficient jumping diffusion 27-point 256^3 (jump 1e6, 32^3 blocks), "
           "PCG + K-cycle to 1e-8", 27, 256, 256, 256, 1e6, 0.5, "pcg"),
    "c5": ("3D 7-point Poisson 512^3 (134M unknowns), PCG + K-cycle to 1e-8", 3, 512, 512, 512,
           1.0, 0.5, "pcg"),
}
JUMP_BLOCK = 32  # c4: coefficient jump on a checkerboard of 32^3 blocks
PROF_SMOOTH, PROF_SPMV = 1, 2
METRIC = "setup+solve DOF/s"


def load_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic():
    p = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.t0 = self.t1 = None

    def __enter__(self):
        if os.environ.get("AGGMG_BENCH_NO_CLOCKS") == "1":  # diagnosis only
            self.t0 = time.time()
            return self
        # started ahead of the timed region (nvidia-smi's own start-up takes driver time that
        # would otherwise land in the first timed step); samples outside [t0, t1] are dropped
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(1.0)
        except OSError:
            self.proc = None
        self.t0 = time.time()
        return self

    def __exit__(self, *a):
        self.t1 = time.time()
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            for ln in out.splitlines():
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    continue
                if self.t0 - 0.25 <= ts <= self.t1 + 0.25:
                    self.lines.append(",".join(parts[1:]))

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Dist:
    def __init__(self, world, local):
        self.world = world
        self.torch = None
        if world > 1:
            import torch
            import torch.distributed as dist

            torch.cuda.set_device(local)
            dist.init_process_group("nccl")
            self.torch, self.dist = torch, dist

    def barrier(self):
        if self.torch:
            self.torch.cuda.synchronize()
            self.dist.barrier()

    def max(self, v):
        if not self.torch:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v):
        if not self.torch:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.torch:
            self.dist.destroy_process_group()


def world_grid_dims(dims, nx, ny, nz, world, scaling="weak"):
    """The global grid at `world` GPUs from a per-GPU grid: weak scaling doubles x, then y, then
    z, a remaining odd factor stacks along the slowest axis; strong scaling keeps
    the grid."""
    if scaling == "strong" or world == 1:
        return nx, ny, nz
    g = [nx, ny, nz]
    axes = [0, 1] if dims == 2 else [0, 1, 2]
    w, i = world, 0
    while w % 2 == 0:
        g[axes[i % len(axes)]] *= 2
        w //= 2
        i += 1
    g[axes[-1]] *= w
    return tuple(g)


def world_grid(cfg_name, world, scaling):
    """The config's global grid at `world` GPUs (weak: 256^3 -> 512x256x256 -> 512x512x256 ->
    512^3 for c2)."""
    label, dims, nx, ny, nz, eps, alpha, method = CONFIGS[cfg_name]
    return world_grid_dims(dims, nx, ny, nz, world, scaling)


def grid_nnz(dims, nx, ny, nz):
    """Stored entries of the generated operators (Dirichlet rows eliminated)."""
    n = nx * ny * nz
    if dims == 27:
        return (3 * nx - 2) * (3 * ny - 2) * (3 * nz - 2)
    if dims == 2:
        return n + 2 * ((nx - 1) * ny + nx * (ny - 1))
    return n + 2 * ((nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1))


def workload_config(cfg_name, world, scaling):
    """The `config` object of the JSON line: identical in the B200 and the reference arms."""
    label, dims, nx, ny, nz, eps, alpha, method = CONFIGS[cfg_name]
    gx, gy, gz = world_grid(cfg_name, world, scaling)
    return {
        "workload": label, "grid": [gx, gy, gz], "n": gx * gy * gz,
        "nnz": grid_nnz(dims, gx, gy, gz),
        "solver": "pcg" if method == "pcg" else "fgmres(30)", "tol": 1e-8,
        "preconditioner": f"hybrid K-cycle AMG (k_levels 2, t 0.25, inner GMRES), alpha {alpha}, "
                          "coarse_size_max 600, damped Jacobi, seed 42",
        "rhs": "b = B0 = ones, x0 = 0",
        "scaling": scaling if world > 1 else "weak",
    }


def configs_c(M, alpha, method, tol=1e-8, max_iters=500):
    setup = M.SetupConfig(alpha=alpha, reuse_caches=True)
    cycle = M.CycleConfig()
    solver = M.SolverConfig(method=M.PCG if method == "pcg" else M.FGMRES, tol=tol,
                            max_iters=max_iters, restart=30)
    return setup, cycle, solver


def reference_matrix(cfg_name, grid):
    """The config's matrix on the host, generated by the reference itself (poisson.cpp) or, for
    the 27-point jump problem that has no reference generator, by the C restatement."""
    from oracle import checkers

    label, dims, nx, ny, nz, eps, alpha, method = CONFIGS[cfg_name]
    gx, gy, gz = grid
    if dims == 27:
        return checkers.oracle().generate_jump27(gx, gy, gz, eps, JUMP_BLOCK)
    return checkers.ref().generate_poisson(2 if dims == 2 else 3, gx, gy, gz, eps)


def cpu_reference_run(M, cfg_name, A, threads, reuse_caches=False):
    """One setup + solve by the reference (oracle/_ref) on all host threads."""
    from oracle import checkers

    label, dims, nx, ny, nz, eps, alpha, method = CONFIGS[cfg_name]
    r = checkers.ref()
    r.lib.fn("set_num_threads")(threads)
    setup, cycle, solver = configs_c(M, alpha, method)
    setup.reuse_caches = reuse_caches
    t0 = time.perf_counter()
    res = r.setup_and_solve(A, np.ones(A.n_rows), setup, cycle, solver)
    return time.perf_counter() - t0, res


def run_reference_arm(args, world, rank):
    """The reference's own CPU implementation on the same configuration (rank 0 only)."""
    from paper_1403_1649_b200 import aggmg as M

    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    dims = CONFIGS[args.config][1]
    grid = world_grid(args.config, args.gpus, args.scaling)
    small = (64, 64, 1) if dims == 2 else (64, 64, 64)
    Aw = reference_matrix(args.config, small)
    for _ in range(args.warmup):
        cpu_reference_run(M, args.config, Aw, threads)
    del Aw
    # The full configuration every step, unless K steps of it cannot finish inside the arm's
    # budget (the weak-scaling grids at 4 and 8 GPUs: 67 M / 134 M unknowns, minutes per step
    # on 16 cores): then the largest grid of the same class that fits, halving the longest axis
    # (the reference's DOF/s barely depends on the size; the line says which grid was timed).
    budget = args.ref_budget_s
    est_rate = 5.0e5 * threads / 16.0  # DOF/s of the reference on this class (c2, 16 cores: 5.9e5)
    sgrid = list(grid)
    while sgrid[0] * sgrid[1] * sgrid[2] * args.steps / est_rate > budget and max(sgrid) > 64:
        sgrid[sgrid.index(max(sgrid))] //= 2
    full = tuple(sgrid) == tuple(grid)
    A = reference_matrix(args.config, tuple(sgrid))
    times = []
    for _ in range(args.steps):
        dt, res = cpu_reference_run(M, args.config, A, threads)
        times.append(dt)
    total = sum(times)
    value = A.n_rows * len(times) / total
    what = (f"the full configuration ({grid[0]}x{grid[1]}x{grid[2]}, {A.n_rows} unknowns)" if full else
            f"a {sgrid[0]}x{sgrid[1]}x{sgrid[2]} grid of the configuration's class ({A.n_rows} unknowns; the "
            f"full {grid[0]}x{grid[1]}x{grid[2]} x {args.steps} steps exceeds the {budget:.0f} s arm budget)")
    sample = (f"{what} every timed step: "
              f"setup_hierarchy + {'pcg' if CONFIGS[args.config][7] == 'pcg' else 'fgmres'} to 1e-8 "
              f"({res.report.iterations} iterations), the reference's default Galerkin path "
              f"(reuse_caches = false, its faster one); warm-up steps on a 64^{2 if dims == 2 else 3} grid")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DOF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": args.scaling if args.gpus > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.config, args.gpus, args.scaling),
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "detail": {"timed_grid": sgrid, "full_configuration": full,
                   "step_seconds": times, "iterations": res.report.iterations,
                   "setup_seconds": res.report.setup_seconds,
                   "solve_seconds": res.report.solve_seconds},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_b200(args, world, rank, local):
    from paper_1403_1649_b200 import _abi
    from paper_1403_1649_b200 import aggmg as M

    dist = Dist(world, local)
    gpu = M.b200()
    lib = gpu.lib
    if lib.fn("init")(local) != 0:
        raise RuntimeError(lib.fn("last_error")().decode())

    def check(rc):
        if rc != 0:
            raise RuntimeError(lib.fn("last_error")().decode())

    label, dims, nx, ny, nz, eps, alpha, method = CONFIGS[args.config]
    setup, cycle, solver = configs_c(M, alpha, method)
    s_c, c_c, v_c = setup._c(), cycle._c(), solver._c()

    dm = C.c_void_p()
    if dims == 27:
        check(lib.fn("dmatrix_jump27")(nx, ny, nz, eps, JUMP_BLOCK, C.byref(dm)))
    else:
        check(lib.fn("dmatrix_poisson")(dims, nx, ny, nz, eps, -1, C.byref(dm)))
    n_, nnz_ = C.c_int64(), C.c_int64()
    check(lib.fn("dmatrix_size")(dm, C.byref(n_), C.byref(nnz_)))
    sell_ = C.c_int32()
    check(lib.fn("dmatrix_format")(dm, C.byref(sell_)))
    l0_sell = bool(sell_.value)
    l0_vi = sell_.value == 2  # SELL-32 with the one-byte value dictionary
    l0_pat = sell_.value == 3  # the row-pattern dictionary (two bytes per row)
    n, nnz = n_.value, nnz_.value
    hist = np.zeros(solver.max_iters + 2)

    def step(record):
        h = C.c_void_p()
        check(lib.fn("setup_hierarchy_device")(dm, C.byref(s_c), C.byref(h)))
        rep = _abi.SolveReportC()
        rep.history = hist.ctypes.data_as(_abi.f64p)
        rep.history_capacity = hist.shape[0]
        check(lib.fn("solve_device")(h, C.byref(c_c), C.byref(v_c), None, C.byref(rep)))
        if record is not None:
            sms = C.c_double()
            check(lib.fn("hierarchy_setup_ms")(h, C.byref(sms)))
            record.append({"setup_ms": sms.value, "solve_s": rep.solve_seconds,
                           "iterations": rep.iterations, "converged": bool(rep.converged),
                           "levels": int(lib.fn("hierarchy_n_levels")(h))})
        lib.fn("hierarchy_free")(h)

    for _ in range(args.warmup):
        step(None)

    # ---- timed region: value (inputs resident in HBM) ----
    records = []
    if not args.no_prof:
        check(lib.fn("profile_enable")((1 << PROF_SMOOTH) | (1 << PROF_SPMV)))
    launches0 = lib.fn("kernel_launches")()
    dist.barrier()
    check(lib.fn("synchronize")())
    with ClockSampler(local) as clk:
        check(lib.fn("timer_start")())
        for _ in range(args.steps):
            step(records)
        ms = C.c_double()
        check(lib.fn("timer_stop")(C.byref(ms)))
    dist.barrier()
    launches = lib.fn("kernel_launches")() - launches0
    elapsed_ms = dist.max(ms.value)
    total_dof = dist.sum(float(n * args.steps))
    value = total_dof / (elapsed_ms / 1e3)

    fam = {}
    for f, name in ((PROF_SMOOTH, "jacobi_l0"), (PROF_SPMV, "spmv_l0")):
        t, cnt, by = C.c_double(), C.c_int64(), C.c_double()
        check(lib.fn("profile_read")(f, C.byref(t), C.byref(cnt), C.byref(by)))
        fam[name] = (t.value, cnt.value, by.value)
    check(lib.fn("profile_enable")(0))

    # ---- end to end through the host C-ABI (host CSR in, x out) ----
    e2e = None
    if not args.no_e2e:
        Ah = (gpu.generate_jump27(nx, ny, nz, eps, JUMP_BLOCK) if dims == 27
              else gpu.generate_poisson(dims, nx, ny, nz, eps))
        b = np.ones(n)
        gpu.setup_and_solve(Ah, b, setup, cycle, solver)  # warm-up
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            res = gpu.setup_and_solve(Ah, b, setup, cycle, solver)
        dt = dist.max(time.perf_counter() - t0)
        h2d = (Ah.row_offsets.nbytes + Ah.col_indices.nbytes + Ah.values.nbytes + b.nbytes)
        e2e = {"value": dist.sum(float(n * args.e2e_steps)) / dt, "unit": "DOF/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(n * 8),
               "iterations": res.report.iterations}
        del Ah

    # ---- e2e through the reference's own call sequence (setup_hierarchy(A, B0)
    # then pcg / fgmres(A, b, x0, M)): the matrix crosses the boundary twice, as in the reference
    e2e_ref_api = None
    if not args.no_e2e and world == 1:
        Ah = (gpu.generate_jump27(nx, ny, nz, eps, JUMP_BLOCK) if dims == 27
              else gpu.generate_poisson(dims, nx, ny, nz, eps))
        b = np.ones(n)
        krylov = gpu.pcg if method == "pcg" else gpu.fgmres

        def api_step():
            hh = gpu.setup_hierarchy(Ah, None, setup)
            return krylov(Ah, b, None, hh, cycle, solver)

        api_step()  # warm-up
        t0 = time.perf_counter()
        for _ in range(2):
            res = api_step()
        dt = (time.perf_counter() - t0) / 2
        e2e_ref_api = {"value": n / dt, "unit": "DOF/s", "ms_per_step": 1e3 * dt,
                       "h2d_bytes_per_step": int(2 * (Ah.row_offsets.nbytes + Ah.col_indices.nbytes
                                                      + Ah.values.nbytes) + b.nbytes),
                       "d2h_bytes_per_step": int(n * 8), "iterations": res.report.iterations,
                       "calls": "aggmg_setup_hierarchy + aggmg_pcg/aggmg_fgmres (C-ABI, host arrays)"}
        del Ah

    # ---- side numbers: the step with the level-0 operator in the other formats — plain fp64
    # SELL values (no value dictionary: operators with more than 256 distinct values, variable
    # coefficients) and, for a row-pattern operator, the dictionary SELL-32 copy
    def side_step(switch, note):
        nonlocal dm
        lib.fn(switch)(0)
        dm2 = C.c_void_p()
        if dims == 27:
            check(lib.fn("dmatrix_jump27")(nx, ny, nz, eps, JUMP_BLOCK, C.byref(dm2)))
        else:
            check(lib.fn("dmatrix_poisson")(dims, nx, ny, nz, eps, -1, C.byref(dm2)))
        saved, dm = dm, dm2
        step(None)  # first sighting of each sub-cycle: eager
        step(None)  # second: graph capture
        nrec = []
        check(lib.fn("synchronize")())
        check(lib.fn("timer_start")())
        for _ in range(2):
            step(nrec)
        check(lib.fn("timer_stop")(C.byref(ms)))
        lib.fn(switch)(1)
        dm = saved
        lib.fn("dmatrix_free")(dm2)
        return {"ms_per_step": ms.value / 2, "setup_ms": nrec[0]["setup_ms"],
                "solve_ms": 1e3 * nrec[0]["solve_s"], "iterations": nrec[0]["iterations"],
                "note": note}

    no_dict = sell_dict = None
    if not args.no_exact and world == 1 and (l0_vi or l0_pat):
        no_dict = side_step("set_value_dictionary",
                            "aggmg_set_value_dictionary(0): SELL-32 with 8-byte values, as on a "
                            "variable-coefficient operator; not the headline")
    if not args.no_exact and world == 1 and l0_pat:
        sell_dict = side_step("set_row_patterns",
                              "aggmg_set_row_patterns(0): level 0 as the SELL-32 copy with one-byte "
                              "value codes instead of row patterns; not the headline")

    # ---- side number: the same step in bit-identical mode (aggmg_set_exact_reductions) ----
    exact = None
    if not args.no_exact:
        lib.fn("set_exact_reductions")(1)
        step(None)  # exact mode has its own sub-cycle graphs: eager, then captured
        step(None)
        erec = []
        dist.barrier()
        check(lib.fn("synchronize")())
        check(lib.fn("timer_start")())
        for _ in range(2):
            step(erec)
        check(lib.fn("timer_stop")(C.byref(ms)))
        lib.fn("set_exact_reductions")(0)
        exact = {"ms_per_step": dist.max(ms.value) / 2, "iterations": erec[0]["iterations"],
                 "note": "aggmg_set_exact_reductions(1): residual history and x bit-identical "
                         "to the reference (DESIGN.md section 5); not the headline"}

    # ---- CPU baseline (reference, all host cores, bounded sample) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libaggmg_ref.so")):
        # the reference on the SAME configuration, once per Galerkin path: the default direct
        # R(AP) products (its faster path) and the cached sort/segmented reduce this library
        # reproduces bit for bit (reuse_caches = true)
        threads = os.cpu_count() or 1
        A = reference_matrix(args.config, (nx, ny, nz))
        dt, cres = cpu_reference_run(M, args.config, A, threads, reuse_caches=False)
        dt2, cres2 = cpu_reference_run(M, args.config, A, threads, reuse_caches=True)
        cpu = {"value": n / dt, "unit": "DOF/s", "cores": threads, "kind": "reference",
               "sample": f"one full setup+solve of the configuration ({nx}x{ny}x{nz}) by the reference, "
                         f"default Galerkin path: {dt:.1f} s ({cres.report.setup_seconds:.1f} s setup, "
                         f"{cres.report.iterations} its)",
               "cache_path": {"value": n / dt2, "seconds": dt2,
                              "setup_seconds": cres2.report.setup_seconds,
                              "iterations": cres2.report.iterations,
                              "note": "reuse_caches = true: the summation order the B200 path reproduces"}}
        del A

    peak, peak_src = load_peak()
    jt, jc, jb = fam["jacobi_l0"]
    st, sc_, sb = fam["spmv_l0"]
    roof = None
    if jc > 0:
        achieved = (jb / jc) / ((jt / jc) / 1e3) / 1e9
        if l0_pat:
            tkey = "jacobidot2_pat_l0_dram_bytes_per_launch"
            kname = ("k_pat<Epi::kJacobiDot2> on level 0: the damped-Jacobi post-smoothing sweep "
                     "over the row-pattern copy of the operator (a two-byte pattern id per row; "
                     "offsets and values from the pattern tables) with PCG's two dot products "
                     "(r.z, r_old.z) fused")
        elif l0_vi and dims != 27:
            # short rows (< 10 per row) on a dictionary copy: PCG's (r.z, r_old.z) ride on the sweep
            tkey = "jacobidot2_sell_vi_l0_dram_bytes_per_launch"
            kname = ("k_sell<Epi::kJacobiDot2, VI> on level 0: the damped-Jacobi post-smoothing "
                     "sweep over the SELL-32 copy of the operator (values as one-byte dictionary "
                     "codes) with PCG's two dot products (r.z, r_old.z) fused")
        elif l0_vi:
            tkey = "jacobi_sell_vi_l0_dram_bytes_per_launch"
            kname = ("k_sell<Epi::kJacobi, VI> on level 0: the damped-Jacobi post-smoothing sweep "
                     "over the SELL-32 copy of the operator, values as one-byte dictionary codes")
        elif l0_sell:
            tkey = "jacobi_sell_l0_dram_bytes_per_launch"
            kname = ("k_sell<Epi::kJacobi> on level 0: the damped-Jacobi post-smoothing sweep "
                     "over the SELL-32 copy of the operator")
        else:
            tkey = "jacobidot2_l0_dram_bytes_per_launch"
            kname = ("k_csr_stream<Epi::kJacobiDot2> on level 0: the fused damped-Jacobi "
                     "post-smoothing sweep that also produces PCG's (r.z, r_old.z)")
        traffic = load_traffic().get(args.config, {}).get(tkey)
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": kname,
                "bytes_per_launch": jb / jc, "avg_launch_ms": jt / jc, "launches": jc,
                "peak_source": peak_src,
                "share_of_step": jt / elapsed_ms if world == 1 else None}
    spmv_gbs = (sb / sc_) / ((st / sc_) / 1e3) / 1e9 if sc_ > 0 else None

    r0 = records[0] if records else {}
    line = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic: device-generated " + ("27-point jumping-coefficient matrix (DESIGN.md §7)"
                 if dims == 27 else "Poisson matrix (poisson.cpp semantics)") + ", b = B0 = ones, x0 = 0"),
        "config": workload_config(args.config, 1, "weak"),
        "detail": {"levels": r0.get("levels"),
                   "iterations": r0.get("iterations"), "converged": r0.get("converged"),
                   "setup_ms": statistics.median(r["setup_ms"] for r in records),
                   "solve_ms": 1e3 * statistics.median(r["solve_s"] for r in records),
                   "solve_dof_per_s": n / statistics.median(r["solve_s"] for r in records),
                   "level0_spmv_residual_gbs": spmv_gbs,
                   "galerkin": "cached sort/segmented reduce (reference reuse_caches=true order)",
                   "l2": f"inputs larger than L2 (A alone is {(12 * nnz + 4 * n) / 1e9:.2f} GB)",
                   "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                   "exact_mode": exact, "no_value_dictionary": no_dict,
                   "sell_dictionary_level0": sell_dict,
                   "e2e_reference_call_sequence": e2e_ref_api},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    lib.fn("dmatrix_free")(dm)
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.close()
    return 0


def rank_bench(comm, rank, local, args, sync_max, sync_sum):
    """One rank of the partitioned benchmark (NCCL process or emulated rank thread).
    sync_max / sync_sum reduce a float over the ranks (host)."""
    from paper_1403_1649_b200 import aggmg as M
    from paper_1403_1649_b200 import dist as D

    lib = M.b200().lib
    world = comm.size
    label, dims, nx, ny, nz, eps, alpha, method = CONFIGS[args.config]
    gx, gy, gz = world_grid(args.config, world, args.scaling)
    setup, cycle, solver = configs_c(M, alpha, method)
    if dims == 27:
        dA = D.DistMatrix.jump27(comm, gx, gy, gz, eps, JUMP_BLOCK)
    else:
        dA = D.DistMatrix.poisson(comm, dims, gx, gy, gz, eps)
    n_glob, row0, nloc, nnz_loc = dA.info()
    fmt = C.c_int32()
    lib.fn("dist_matrix_format")(dA._h, C.byref(fmt))
    nnz_glob = sync_sum(float(nnz_loc))

    def step(record):
        h = D.setup(comm, dA, setup, agglomerate_rows=args.agglomerate)
        res = h.solve(solver, cycle)
        if record is not None:
            nl, nd, sms = h.info()
            record.append({"setup_ms": sms, "solve_s": res.report.solve_seconds,
                           "iterations": res.report.iterations, "converged": res.report.converged,
                           "levels": nl, "distributed_levels": nd})
        h.free()

    for _ in range(args.warmup):
        step(None)
    records = []
    if rank == 0 and not args.no_prof:
        lib.fn("profile_enable")((1 << PROF_SMOOTH) | (1 << PROF_SPMV))
    launches0 = lib.fn("kernel_launches")()
    comm.barrier()
    with ClockSampler(local) as clk:
        lib.fn("timer_start")()
        for _ in range(args.steps):
            step(records)
        ms = C.c_double()
        lib.fn("timer_stop")(C.byref(ms))
    comm.barrier()
    launches = lib.fn("kernel_launches")() - launches0
    elapsed_ms = sync_max(ms.value)
    value = n_glob * args.steps / (elapsed_ms / 1e3)
    fam = {}
    if rank == 0:
        for f, name in ((PROF_SMOOTH, "jacobi_l0"), (PROF_SPMV, "spmv_l0")):
            t, cnt, by = C.c_double(), C.c_int64(), C.c_double()
            lib.fn("profile_read")(f, C.byref(t), C.byref(cnt), C.byref(by))
            fam[name] = (t.value, cnt.value, by.value)
        lib.fn("profile_enable")(0)

    # end to end: this rank's host slab in, its part of x out
    e2e = None
    if not args.no_e2e:
        kind = "jump27" if dims == 27 else "poisson"
        rows = D.host_rows(kind, row0, nloc, gx, gy, gz, eps, dims=2 if dims == 2 else 3,
                           jump=eps, block=JUMP_BLOCK)
        b = np.ones(nloc)
        comm.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            A2 = D.DistMatrix.from_rows(comm, n_glob, row0, rows)
            h = D.setup(comm, A2, setup, agglomerate_rows=args.agglomerate)
            res = h.solve(solver, cycle, b_local=b, n_local=nloc)
            h.free()
            A2.free()
        comm.barrier()
        dt = sync_max(time.perf_counter() - t0)
        h2d = rows.row_offsets.nbytes + rows.col_indices.nbytes + rows.values.nbytes + b.nbytes
        e2e = {"value": n_glob * args.e2e_steps / dt, "unit": "DOF/s",
               "h2d_bytes_per_step": int(sync_sum(float(h2d))),
               "d2h_bytes_per_step": int(n_glob * 8), "iterations": res.report.iterations}
    dA.free()
    if rank != 0:
        return None
    peak, peak_src = load_peak()
    roof = None
    jt, jc, jb = fam.get("jacobi_l0", (0, 0, 0))
    if jc > 0:
        achieved = (jb / jc) / ((jt / jc) / 1e3) / 1e9
        kname = {3: "k_pat<Epi::kJacobi> (row-pattern ids)",
                 2: "k_sell<Epi::kJacobi, VI> (SELL-32, one-byte value codes)",
                 1: "k_sell<Epi::kJacobi> (SELL-32)",
                 0: "k_csr_stream<Epi::kJacobi>"}[fmt.value]
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None,
                "kernel": kname + " on level 0: the damped-Jacobi sweep over rank 0's slab",
                "bytes_per_launch": jb / jc, "avg_launch_ms": jt / jc, "launches": jc,
                "peak_source": peak_src, "share_of_step": jt / elapsed_ms}
    r0 = records[0] if records else {}
    return {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic: device-generated " + ("27-point jumping-coefficient matrix"
                 if dims == 27 else "Poisson matrix (poisson.cpp semantics)")
                 + ", one row slab per rank, b = B0 = ones, x0 = 0"),
        "config": workload_config(args.config, world, args.scaling),
        "detail": {"levels": r0.get("levels"), "distributed_levels": r0.get("distributed_levels"),
                   "agglomerate_rows": args.agglomerate,
                   "iterations": r0.get("iterations"), "converged": r0.get("converged"),
                   "setup_ms": statistics.median(r["setup_ms"] for r in records),
                   "solve_ms": 1e3 * statistics.median(r["solve_s"] for r in records),
                   "galerkin": "cached sort/segmented reduce order (bit-identical to one GPU)",
                   "l2": "inputs larger than L2",
                   "parallelism": f"row-partitioned x{world} ({comm.kind})"},
        "roofline": roof, "cpu_baseline": None, "e2e": e2e, "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }


def run_dist(args, world, rank, local):
    """torchrun: one process per GPU, NCCL transport."""
    import torch
    import torch.distributed as tdist

    from paper_1403_1649_b200 import dist as D

    torch.cuda.set_device(local)
    tdist.init_process_group("gloo")
    obj = [D.nccl_unique_id() if rank == 0 else None]
    tdist.broadcast_object_list(obj, src=0)
    comm = D.nccl_comm(rank, world, obj[0], local)

    def red(v, op):
        t = torch.tensor([v], dtype=torch.float64)
        tdist.all_reduce(t, op=op)
        return float(t.item())

    line = rank_bench(comm, rank, local, args, lambda v: red(v, tdist.ReduceOp.MAX),
                      lambda v: red(v, tdist.ReduceOp.SUM))
    if rank == 0:
        print(json.dumps(line), flush=True)
    comm.close()
    tdist.destroy_process_group()
    return 0


def run_emulated(args):
    """R rank threads on one GPU (in-process transport): overhead diagnostic."""
    import threading

    from paper_1403_1649_b200 import dist as D

    R = args.emulate_ranks
    vals, lock, out = {}, threading.Lock(), {}
    bar = threading.Barrier(R)

    def reducer(op):
        def f(v):
            with lock:
                vals.setdefault(op, []).append(v)
            bar.wait()
            res = max(vals[op]) if op == "max" else sum(vals[op])
            bar.wait()
            with lock:
                vals.pop(op, None)
            bar.wait()
            return res
        return f

    def fn(comm, rank):
        line = rank_bench(comm, rank, 0, args, reducer("max"), reducer("sum"))
        if rank == 0:
            out["line"] = line

    D.run_threads(R, fn)
    line = out["line"]
    line["config"]["parallelism"] = f"row-partitioned x{R} rank threads emulated on ONE GPU"
    line["n_gpus"] = 1
    print(json.dumps(line), flush=True)
    return 0


def spawn_ranks(n):
    """`python bench.py --gpus N` without a launcher: start N ranks through torch.distributed.run
    on this node (127.0.0.1, a free port); rank 0 prints the JSON line to our stdout."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_dry(args, world, rank):
    """Launcher / rendezvous check on CPU: every rank joins a gloo group, the ranks agree on the
    global grid, and rank 0 prints a config-only line."""
    import torch
    import torch.distributed as tdist

    if world > 1:
        tdist.init_process_group("gloo")
    grid = world_grid(args.config, world, args.scaling)
    rows = grid[0] * grid[1] * grid[2]
    t = torch.tensor([float(rows // world + (1 if rank < rows % world else 0))], dtype=torch.float64)
    if world > 1:
        tdist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "n_gpus": world, "dry_run": True,
                          "rows_covered": int(t.item()), "scaling": args.scaling,
                          "config": workload_config(args.config, world, args.scaling)}), flush=True)
    if world > 1:
        tdist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-exact", action="store_true", help="skip the bit-identical-mode side number")
    ap.add_argument("--no-prof", action="store_true", help="skip per-launch CUDA-event timing")
    ap.add_argument("--ref-budget-s", type=float, default=1400.0,
                    help="--impl reference: seconds the timed steps may take; larger configurations "
                         "time a same-class sample grid instead")
    ap.add_argument("--mode", default="auto", choices=["auto", "single", "dist", "replicas"],
                    help="auto: one GPU -> single, torchrun N>1 -> dist (row-partitioned)")
    ap.add_argument("--agglomerate", type=int, default=0,
                    help="rows at or below which a level is gathered on rank 0 (0 = default)")
    ap.add_argument("--emulate-ranks", type=int, default=0)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak keeps the config's problem per GPU, strong keeps its grid")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check without a GPU: ranks rendezvous over gloo, agree on the "
                         "workload and print the config line (tests/test_bench_launcher.py)")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if (args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200"
            and args.emulate_ranks == 0 and args.mode != "replicas"):
        return spawn_ranks(args.gpus)  # one process per GPU, like the driver's torchrun
    # Native libraries (NCCL's version banner, driver messages) write to fd 1; point fd 1 at
    # stderr and keep the real stdout for the JSON line alone.
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    sys.stdout.flush()
    real_stdout = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(real_stdout, "w", buffering=1)
    if args.dry_run:
        return run_dry(args, world, rank)
    if args.impl == "reference":
        return run_reference_arm(args, world, rank)
    if args.emulate_ranks > 0:
        return run_emulated(args)
    mode = args.mode
    if mode == "auto":
        mode = "dist" if world > 1 else "single"
    if mode == "dist":
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        return run_dist(args, world, rank, local)
    return run_b200(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
