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

Multi-GPU (torchrun, --gpus N > 1): the ROW-PARTITIONED solver: the grid of
the config is stacked N times along its slowest axis (weak scaling, the config's problem per
GPU), each rank generates and owns one slab, setup and solve exchange halos and scalars over
NCCL, coarse levels are agglomerated on rank 0.  --mode replicas instead runs N independent
copies; --emulate-ranks R runs the partitioned path as R rank threads on one GPU (a
transport/overhead diagnostic, not a scaling number).
--impl reference times the reference CPU implementation on the host cores instead.
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


def configs_c(M, alpha, method, tol=1e-8, max_iters=500):
    setup = M.SetupConfig(alpha=alpha, reuse_caches=True)
    cycle = M.CycleConfig()
    solver = M.SolverConfig(method=M.PCG if method == "pcg" else M.FGMRES, tol=tol,
                            max_iters=max_iters, restart=30)
    return setup, cycle, solver


def cpu_reference_run(M, cfg_name, sample_n, threads):
    """One setup+solve of the reference (oracle/_ref) on a bounded sample grid."""
    label, dims, nx, ny, nz, eps, alpha, method = CONFIGS[cfg_name]
    from oracle import checkers

    r = checkers.ref()
    r.lib.fn("set_num_threads")(threads)
    if dims == 27:
        A = checkers.oracle().generate_jump27(sample_n, sample_n, sample_n, eps, JUMP_BLOCK)
    elif dims == 3:
        A = r.generate_poisson(3, sample_n, sample_n, sample_n, eps)
    else:
        A = r.generate_poisson(2, sample_n, sample_n, 1, eps)
    setup, cycle, solver = configs_c(M, alpha, method)
    setup.reuse_caches = False  # the reference's default (faster) Galerkin path
    t0 = time.perf_counter()
    res = r.setup_and_solve(A, np.ones(A.n_rows), setup, cycle, solver)
    dt = time.perf_counter() - t0
    return A.n_rows, dt, res


def run_reference_arm(args, world, rank):
    from paper_1403_1649_b200 import aggmg as M

    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    dims = CONFIGS[args.config][1]
    sample_n = args.ref_sample or (512 if dims == 2 else (64 if dims == 27 else 96))
    times, n = [], 0
    for i in range(args.warmup + args.steps):
        n, dt, res = cpu_reference_run(M, args.config, sample_n, threads)
        if i >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = n * len(times) / total
    sample = (f"{sample_n}^{2 if dims == 2 else 3} grid of the same problem class, full setup+solve per step "
              f"(reference default Galerkin path), {res.report.iterations} iterations")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DOF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CONFIGS[args.config][0], "sample": sample},
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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

    # ---- side number: the same step in bit-identical mode (aggmg_set_exact_reductions) ----
    exact = None
    if not args.no_exact:
        lib.fn("set_exact_reductions")(1)
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
        threads = os.cpu_count() or 1
        sample_n = 512 if dims == 2 else (96 if dims == 27 else 128)
        ns, dt, cres = cpu_reference_run(M, args.config, sample_n, threads)
        cpu = {"value": ns / dt, "unit": "DOF/s", "cores": threads, "kind": "reference",
               "sample": f"one setup+solve of the {sample_n}^{2 if dims == 2 else 3} grid (reference default "
                         f"Galerkin path, {cres.report.iterations} its, {dt:.1f} s)"}

    peak, peak_src = load_peak()
    jt, jc, jb = fam["jacobi_l0"]
    st, sc_, sb = fam["spmv_l0"]
    roof = None
    if jc > 0:
        achieved = (jb / jc) / ((jt / jc) / 1e3) / 1e9
        if l0_vi:
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
        "config": {"workload": label, "n": n, "nnz": nnz, "levels": r0.get("levels"),
                   "iterations": r0.get("iterations"), "converged": r0.get("converged"),
                   "setup_ms": statistics.median(r["setup_ms"] for r in records),
                   "solve_ms": 1e3 * statistics.median(r["solve_s"] for r in records),
                   "solve_dof_per_s": n / statistics.median(r["solve_s"] for r in records),
                   "level0_spmv_residual_gbs": spmv_gbs,
                   "galerkin": "cached sort/segmented reduce (reference reuse_caches=true order)",
                   "l2": f"inputs larger than L2 (A alone is {(12 * nnz + 4 * n) / 1e9:.2f} GB)",
                   "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                   "exact_mode": exact},
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


def dist_grid(dims, nx, ny, nz, world):
    """Weak scaling: the config's grid per rank, stacked along the slowest axis."""
    if dims == 2:
        return nx, ny * world, 1
    return nx, ny, nz * world


def rank_bench(comm, rank, local, args, sync_max, sync_sum):
    """One rank of the partitioned benchmark (NCCL process or emulated rank thread).
    sync_max / sync_sum reduce a float over the ranks (host)."""
    from paper_1403_1649_b200 import aggmg as M
    from paper_1403_1649_b200 import dist as D

    lib = M.b200().lib
    world = comm.size
    label, dims, nx, ny, nz, eps, alpha, method = CONFIGS[args.config]
    gx, gy, gz = dist_grid(dims, nx, ny, nz, world)
    setup, cycle, solver = configs_c(M, alpha, method)
    if dims == 27:
        dA = D.DistMatrix.jump27(comm, gx, gy, gz, eps, JUMP_BLOCK)
    else:
        dA = D.DistMatrix.poisson(comm, dims, gx, gy, gz, eps)
    n_glob, row0, nloc, nnz_loc = dA.info()
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
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None,
                "kernel": "k_csr_stream<Epi::kJacobi> on level 0 (rank 0's slab)",
                "bytes_per_launch": jb / jc, "avg_launch_ms": jt / jc, "launches": jc,
                "peak_source": peak_src, "share_of_step": jt / elapsed_ms}
    r0 = records[0] if records else {}
    return {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic: device-generated " + ("27-point jumping-coefficient matrix"
                 if dims == 27 else "Poisson matrix (poisson.cpp semantics)")
                 + ", one row slab per rank, b = B0 = ones, x0 = 0"),
        "config": {"workload": label + f" per GPU, stacked x{world} along the slowest axis",
                   "grid": [gx, gy, gz], "n": n_glob, "nnz": int(nnz_glob),
                   "levels": r0.get("levels"), "distributed_levels": r0.get("distributed_levels"),
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
    ap.add_argument("--ref-sample", type=int, default=0)
    ap.add_argument("--mode", default="auto", choices=["auto", "single", "dist", "replicas"],
                    help="auto: one GPU -> single, torchrun N>1 -> dist (row-partitioned)")
    ap.add_argument("--agglomerate", type=int, default=0,
                    help="rows at or below which a level is gathered on rank 0 (0 = default)")
    ap.add_argument("--emulate-ranks", type=int, default=0)
    args = ap.parse_args()
    # Native libraries (NCCL's version banner, driver messages) write to fd 1; point fd 1 at
    # stderr and keep the real stdout for the JSON line alone.
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    sys.stdout.flush()
    real_stdout = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(real_stdout, "w", buffering=1)
    world, rank, local = dist_env()
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
